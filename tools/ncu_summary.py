"""Write profiles/ncu_summary.json (+ a text summary) from one `ncu --set full` capture of sim_kernel.

usage: python tools/ncu_summary.py REPORT.ncu-rep TAG "capture description" INSTANCES ALG_BYTES [KERNEL] [REQUESTS]
ALG_BYTES = SURVEY §8(d) algorithmic bytes of the captured launch (bench.py prints alg_bytes_per_launch).
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, tag, capture, inst, alg = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), float(sys.argv[5])
kernel = sys.argv[6] if len(sys.argv) > 6 else "slosim::sim_kernel"
requests = int(sys.argv[7]) if len(sys.argv) > 7 else None
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
num = lambda k: float(d[k].replace(",", ""))
keep = ["launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: num(k) for k in d
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(stalls.values()) or 1.0
dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
unit = rows[1][rows[0].index("dram__bytes_read.sum")]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
dram *= scale
out = {
    "round": 2, "tag": tag, "kernel": kernel, "capture": capture, "launch_instances": inst, "instances": inst,
    "gpu_time_ms_under_ncu": num("gpu__time_duration.sum") * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                                                                 "s": 1e3, "second": 1e3}.get(rows[1][rows[0].index("gpu__time_duration.sum")], 1.0),
    "dram_bytes_per_launch": dram, "alg_bytes_per_launch": alg, "dram_over_alg": dram / alg,
    "dram_bytes_per_instance": dram / inst, "alg_bytes_per_instance": alg / inst,
    "metrics": {k: d[k] for k in keep if k in d},
    "stall_breakdown_pct": {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if v > 0},
    "warp_inst_per_request": num("smsp__inst_executed.sum") / requests if requests else None,
}
with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
    json.dump(out, f, indent=1)
txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_report.py"), rep, "40"],
                     capture_output=True, text=True).stdout
with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_{kernel.split('::')[-1]}.txt"), "w") as f:
    f.write(txt)
print(json.dumps(out, indent=1))
