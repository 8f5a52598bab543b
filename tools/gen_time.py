"""Time device trace generation (slosim_gen_longtail) vs numpy on the host for each config's traces."""
import json
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402

out = {}
for name in ("config1", "config2", "config4", "config5"):
    r = bench.trace_generation(name)
    out[name] = r
    print(name, json.dumps(r), flush=True)
