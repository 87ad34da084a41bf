"""Opcode histogram of the hottest backward-branch loop of one kernel in a
cuobjdump -sass dump: python tools/sass_loop.py dump.sass <name-substring> [lo hi]."""
import collections, re, sys
s = open(sys.argv[1]).read()
for f in s.split('Function : ')[1:]:
    if sys.argv[2] not in f.split('\n')[0]:
        continue
    ins = [(int(a, 16), t.strip()) for a, t in re.findall(r'/\*([0-9a-f]{4,5})\*/\s+([^;]*);', f)]
    loops = []
    for a, t in ins:
        m = re.search(r'BRA (0x[0-9a-f]+)', t)
        if m and int(m.group(1), 16) < a:
            loops.append((a - int(m.group(1), 16), int(m.group(1), 16), a))
    if len(sys.argv) > 4:
        lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
    else:
        _, lo, hi = max(loops)
    body = [t for a, t in ins if lo <= a <= hi]
    c = collections.Counter(re.sub(r'^@!?U?P\w+\s+', '', t).split(' ')[0].split('.')[0] for t in body)
    print(f"{f.split(chr(10))[0][:100]}\nloop {lo:#x}-{hi:#x}: {len(body)} instructions")
    for op, n in c.most_common(25):
        print(f"  {op:10s} {n}")
    break
