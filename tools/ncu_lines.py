"""Per-source-line instruction and stall-sample totals of one launch in an
ncu report (`--page source --print-source cuda,sass`)."""
import collections, csv, io, subprocess, sys
rep, skip = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
n_show = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(skip), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
cur = None; agg = collections.Counter(); samp = collections.Counter(); text = {}; fname = ''
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == 'File Path':
        fname = r[1].split('/')[-1]; continue
    if len(r) < 8 or r[0] == 'Line No':
        continue
    if r[0] and r[0] != '-' and r[0].isdigit():
        cur = (fname, int(r[0])); text[cur] = r[1][:80]
    try:
        n = float(r[7].replace(',', '')); s = float(r[4].replace(',', ''))
    except ValueError:
        continue
    agg[cur] += n; samp[cur] += s
tot = sum(agg.values()) or 1; ts = sum(samp.values()) or 1
print(f"warp-instructions {tot:.3e}, stall samples {ts:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -samp[kv[0]])[:n_show]:
    print(f"{v:10.3e} {100*v/tot:5.1f}%  stall {100*samp[k]/ts:5.1f}%  {k[0]}:{k[1]} {text.get(k, '')}")
