"""Write a text summary of an ncu --set full report (per launch) + DRAM traffic JSON."""
import csv, io, json, subprocess, sys
rep, out_txt = sys.argv[1], sys.argv[2]
out_json = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
want = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_lsu.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg"]
lines = []
traffic = []
for r in data:
    d = {}
    for k in want:
        if k in ix:
            d[k] = r[ix[k]]
    lines.append("\n".join(f"  {k:62s} {v} {units[ix[k]] if k in ix else ''}" for k, v in d.items()))
    try:
        rd = float(d.get("dram__bytes_read.sum", "0").replace(",", ""))
        wr = float(d.get("dram__bytes_write.sum", "0").replace(",", ""))
        ur = units[ix["dram__bytes_read.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ur, 1)
        traffic.append((rd + wr) * scale)
    except Exception:
        pass
with open(out_txt, "w") as f:
    f.write(f"ncu --set full summary of {rep}\n")
    for i, l in enumerate(lines):
        f.write(f"launch {i}:\n{l}\n")
if out_json and traffic:
    json.dump({"source": rep, "kernel": "k_pix_fast<11,11>", "dram_bytes_per_launch": sum(traffic) / len(traffic),
               "per_launch": traffic}, open(out_json, "w"), indent=1)
print(open(out_txt).read()[:3000])
