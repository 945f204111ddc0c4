"""Summarise an ncu --set full report of the apply kernel into profiles/ncu_summary_r01.json
(dram bytes per launch for bench.py's roofline.traffic, plus the headline metrics)."""
import csv, io, json, subprocess, sys

rep, key, out = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "launch__shared_mem_per_block_dynamic",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
launches = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if "apply_dmma" not in d.get("Kernel Name", ""):
        continue
    m = {}
    for w in want:
        if w in d:
            try:
                v = float(d[w].replace(",", ""))
            except ValueError:
                continue
            u = units[hdr.index(w)]
            if u in ("Mbyte", "MB"): v *= 1e6
            elif u in ("Gbyte", "GB"): v *= 1e9
            elif u in ("Kbyte", "KB"): v *= 1e3
            elif u == "msecond": v *= 1e-3
            elif u == "usecond": v *= 1e-6
            elif u == "nsecond": v *= 1e-9
            elif u == "second": pass
            m[w] = v
    m["kernel"] = d.get("Kernel Name")
    launches.append(m)
try:
    summ = json.load(open(out))
except (OSError, ValueError):
    summ = {}
L = launches[-1]
L["dram_bytes_per_launch"] = L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
L["source"] = rep
summ[key] = L
json.dump(summ, open(out, "w"), indent=1)
print(json.dumps(L, indent=1))
