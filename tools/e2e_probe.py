"""Where the host-buffer entry point spends its time (GPU box): wall time of slosim_run_batch_host vs its
own kernel-event time, on config5 slices."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_02329_b200 import _abi
from paper_2605_02329_b200.batch import config5
from paper_2605_02329_b200.pack import PackedBatch

SL = 16384
sw = config5(select=np.arange(0, 4 * SL))
pk = sw.packed
pin = lambda a: torch.from_numpy(np.array(a, copy=True)).pin_memory().numpy()
arr, inp, out, hit, idr = pin(pk.arrival), pin(pk.inp), pin(pk.out), pin(pk.hit), pin(pk.idr)
for s in range(4):
    inst = pin(pk.instances[s * SL:(s + 1) * SL].view(np.uint8)).view(_abi.instance_dtype())
    part = PackedBatch(arr, inp, out, hit, idr, pk.profiles, inst, 0, 0, 0)
    part.summaries = pin(part.summaries.view(np.uint8)).view(_abi.summary_dtype())
    b = part.host_struct()
    ms = ctypes.c_float(0)
    t0 = time.perf_counter()
    rc = _abi.lib().slosim_run_batch_host(ctypes.byref(b), ctypes.byref(ms))
    wall = (time.perf_counter() - t0) * 1e3
    print(f"slice {s}: wall {wall:.1f} ms, kernel events {ms.value:.1f} ms, overhead {wall - ms.value:.1f} ms", flush=True)
