"""Summarise an ncu report: key raw metrics + hottest source lines (by stall samples and instructions)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "launch__grid_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
for i, h in enumerate(hdr):
    if h in want:
        print(f"{h:70s} {units[i]:10s} {vals[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
out, fname = [], None
for r in csv.reader(src.splitlines()):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        try:
            out.append((float(r[7] or 0), float(r[4] or 0), fname, int(r[0]), r[1][:95]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1; ts = sum(o[1] for o in out) or 1
print(f"total inst {tot:.3e}  stall samples {ts:.0f}")
for o in sorted(out, key=lambda x: -x[1])[:top]:
    print(f"{o[0]/tot*100:5.1f}%i {o[1]/ts*100:5.1f}%s {o[2]}:{o[3]} {o[4]}")
