"""Key metrics + top stall reasons of every kernel in an ncu --set full report,
as JSON (dev tool; the summaries under profiles/ come from it).
usage: python tools/ncu_summary.py report.ncu-rep "workload text" > out.json"""
import csv, json, subprocess, sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
rep, workload = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
res = []
for v in rows[2:]:
    m = {n: v[i] for i, n in enumerate(h) if n in WANT}
    u = {n: units[i] for i, n in enumerate(h) if n in WANT}
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
            try:
                st.append((float(v[i]), n[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    m["top_stalls"] = [n for _, n in sorted(st, reverse=True)[:6]]
    res.append({"kernel": v[h.index("Kernel Name")], "metrics": m, "units": u})
print(json.dumps({"report": rep, "workload": workload, "kernels": res}, indent=1))
