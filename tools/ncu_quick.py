"""Key raw metrics and stall split of one kernel in an ncu report: python tools/ncu_quick.py REP [KERNEL_SUBSTR]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if want and want not in d.get("Kernel Name", ""):
        continue
    u = dict(zip(hdr, units))
    keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__t_sector_hit_rate.pct",
            "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
            "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum",
            "lts__t_sectors.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__warps_eligible.avg.per_cycle_active"]
    print(d.get("Kernel Name", "")[:80])
    for k in keys:
        if k in d:
            print(f"  {k:60s} {d[k]:>18s} {u[k]}")
    st = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: float(d[k].replace(",", "")) for k in d
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(st.values()) or 1
    print("  stalls: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
