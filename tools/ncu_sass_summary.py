"""Summarise an `ncu --page source --csv --print-source=sass` dump:
instructions executed and stall samples per opcode, top stall reasons,
and the hottest address ranges."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def num(r, k):
    try: return float(r[ix[k]].replace(',', ''))
    except Exception: return 0.0
by_op = collections.Counter(); samp_op = collections.Counter(); tot = 0; tots = 0
stall_cols = [h for h in hdr if h.startswith('stall_')]
stalls = collections.Counter()
hot = []
for r in data:
    src = r[ix['Source']].strip()
    op = re.sub(r'^@!?U?P\w+\s+', '', src).split(' ')[0] if src else '?'
    n = num(r, 'Instructions Executed'); s = num(r, 'Warp Stall Sampling (All Samples)')
    by_op[op] += n; samp_op[op] += s; tot += n; tots += s
    for c in stall_cols: stalls[c] += num(r, c)
    hot.append((s, r[ix['Address']], src[:60], n))
print(f"total warp-instructions executed {tot:.3e}, stall samples {tots:.0f}")
print("top opcodes by executed instructions:")
for op, n in by_op.most_common(18):
    print(f"  {op:14s} {n:12.3e} {100*n/tot:5.1f}%   samples {100*samp_op[op]/max(tots,1):5.1f}%")
print("stall reasons (samples):")
st = sum(stalls.values()) or 1
for c, v in stalls.most_common(10):
    print(f"  {c:32s} {100*v/st:5.1f}%")
if len(sys.argv) > 2:
    hot.sort(reverse=True)
    for s, a, src, n in hot[:int(sys.argv[2])]:
        print(f"  {a} {s:8.0f} {n:10.3e}  {src}")
