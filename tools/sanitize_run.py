"""Small engine workload for compute-sanitizer: config-1 instances (both pairs) in the throughput and the
row/trace specialisations, a slice of the fuzz sweep (memory mode, table LUTs, noise), a traced Simulation,
and the same small batches forced through the lane engine."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

from paper_2605_02329_b200 import _abi
from paper_2605_02329_b200.batch import config1, run_batch
import test_gpu_fuzz as F

s = run_batch(config1().packed)
assert np.all(s["status"] == 0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
packed = F._batch(flags=_abi.F_ROWS, n_inst=N, seed=5)
run_batch(packed)
packed = F._batch(flags=0, n_inst=N, seed=6)
run_batch(packed)
import paper_2605_02329_b200 as slosim
from paper_2605_02329_b200.workload import LongTailSpec, gen_longtail
wl = gen_longtail(LongTailSpec(n_requests=200))
sim = slosim.Simulation(slosim.ClusterConfig(prefill_policy="kairos-urgency", decode_policy="kairos-slack"), wl,
                        collect_events=True)
sim.run()
# the lane engine (one instance per thread), forced onto small batches: config 1 and a fuzz slice
# (cooperative prefill starts, deferral of out-of-scope instances to the warp engine)
os.environ["SLOSIM_FORCE_LANE_ENGINE"] = "1"
s = run_batch(config1().packed)
assert np.all(s["status"] == 0)
run_batch(F._batch(flags=0, n_inst=N, seed=7))
del os.environ["SLOSIM_FORCE_LANE_ENGINE"]
print("sanitize_run ok")
