#!/bin/bash
# On the GPU box: bench every gpuvar/*.so (plus the in-tree library as "base"),
# print ms_per_step / K2 ms / per-step times.  Extra args go to bench.py.
run() {
  python bench.py --no-cpu-baseline --no-e2e --extras "" "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
x=d.get('extra_configs',{})
print('%-14s ms/step %.4f  k2 %.4f frac %.4f  steps %s k2 %s' % ('$tag', d['ms_per_step'], d['roofline']['k2_ms'], d['roofline']['frac'], d['workload_detail']['step_ms'][:3], d['workload_detail']['k2_step_ms'][:3]), {k:(round(v['ms_per_iteration'],2), round(v.get('k2_ms',0),3), round(v.get('k3_ms',0),2)) for k,v in x.items()})
"
}
tag=base; run "$@"
for so in gpuvar/*.so; do
  [ -e "$so" ] || continue
  tag=$(basename $so .so); PXST_LIB=$PWD/$so run "$@"
done
tag=base2; run "$@"
