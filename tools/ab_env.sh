#!/bin/bash
# On the GPU box: A/B one environment switch of the library on the headline
# bench (alternating runs):  tools/ab_env.sh VAR=VALUE [bench args]
kv=$1; shift
run() {
  env "$@" python bench.py --no-cpu-baseline --no-e2e --extras "${EXTRAS-}" $ARGS 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
x=d.get('extra_configs',{})
print('%-16s ms/step %.4f  k2 %.4f frac %.4f  steps %s' % ('$tag', d['ms_per_step'], d['roofline']['k2_ms'], d['roofline']['frac'], d['workload_detail']['step_ms'][:3]), {k:(round(v['ms_per_iteration'],2), round(v.get('k2_ms',0),3), round(v.get('k3_ms',0),2)) for k,v in x.items()})
"
}
ARGS="$*"
for i in 1 2; do
  tag=default; run A=1
  tag=$kv; run $kv
done
