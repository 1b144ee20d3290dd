"""Summarise an ncu report (raw metrics + top source lines) into profiles/."""
import csv, json, subprocess, sys
rep, out_txt = sys.argv[1], sys.argv[2]
traffic_json = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"]
d = {}
for k in keys:
    if k in hdr:
        i = hdr.index(k)
        d[k] = (vals[i], units[i])
with open(out_txt, "w") as f:
    f.write(f"ncu --set full report: {rep}\n")
    for k, (v, u) in d.items():
        f.write(f"{k:75s} {v} {u}\n")
if traffic_json:
    def num(k):
        v, u = d[k]
        v = float(v.replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    t = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    inst = num("smsp__inst_executed.sum")
    dv, du = d["gpu__time_duration.sum"]
    dur_s = float(dv.replace(",", "")) * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6,
                                          "ms": 1e-3, "msecond": 1e-3}.get(du, 1e-6)
    # issue ceiling: 148 SMs x 4 schedulers x 1 warp instruction per cycle at 1965 MHz
    issue_peak = 148 * 4 * 1965e6
    nveh = int(sys.argv[4]) if len(sys.argv) > 4 else 2000000
    json.dump({"workload": "C4", "n_vehicles": nveh, "kernel": "k_step",
               "dram_bytes_per_launch": t, "warp_inst_per_launch": inst,
               "issue_frac": inst / dur_s / issue_peak,
               "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
               "report": rep}, open(traffic_json, "w"), indent=1)
print(open(out_txt).read())
