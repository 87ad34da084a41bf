"""Decode the control bits (stall count, yield, scoreboards) of a kernel's
SASS from `cuobjdump -sass` and sum the fixed stall cycles over an address
range: python tools/sass_stalls.py dump.sass <name-substring> lo hi."""
import collections, re, sys
s = open(sys.argv[1]).read()
for f in s.split('Function : ')[1:]:
    if sys.argv[2] not in f.split('\n')[0]:
        continue
    lines = f.split('\n')
    lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
    recs = []
    for i, l in enumerate(lines):
        m = re.match(r'\s+/\*([0-9a-f]{4,5})\*/\s+([^;]*);\s+/\* (0x[0-9a-f]+) \*/', l)
        if not m:
            continue
        a = int(m.group(1), 16)
        m2 = re.search(r'/\* (0x[0-9a-f]+) \*/', lines[i + 1])
        hw = int(m2.group(1), 16)
        stall = (hw >> 41) & 0xf
        yld = (hw >> 45) & 1
        wb = (hw >> 46) & 7
        rb = (hw >> 49) & 7
        wmask = (hw >> 52) & 0x3f
        if lo <= a <= hi:
            recs.append((a, m.group(2).strip(), stall, yld, wb, rb, wmask))
    tot = sum(r[2] for r in recs)
    by = collections.Counter(); cnt = collections.Counter()
    for r in recs:
        op = re.sub(r'^@!?U?P\w+\s+', '', r[1]).split(' ')[0].split('.')[0]
        by[op] += r[2]; cnt[op] += 1
    print(f"{len(recs)} instructions, sum of stall counts {tot}")
    for op, v in by.most_common(12):
        print(f"  {op:8s} n={cnt[op]:4d} stall cycles {v:5d} ({v/cnt[op]:.2f} avg)")
    if len(sys.argv) > 5:
        for r in recs[:int(sys.argv[5])]:
            print(f"  {r[0]:05x} s{r[2]} y{r[3]} wb{r[4]} rb{r[5]} w{r[6]:02x}  {r[1][:70]}")
    break
