import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from paper_2605_02329_b200.batch import config1, DeviceBatch
from helpers import pack_config1
a = config1().packed
b, _ = pack_config1()
print("profiles equal", bytes(a.profiles) == bytes(b.profiles), len(bytes(a.profiles)))
print("instances equal", a.instances.tobytes() == b.instances.tobytes())
for k in ("arrival", "inp", "out", "hit", "idr"):
    print(k, np.array_equal(getattr(a, k), getattr(b, k)), getattr(a, k).dtype, getattr(a, k).shape, getattr(b,k).shape)
for name, pk in (("grid", a), ("builder", b)):
    db = DeviceBatch(pk)
    print(name, "dev profiles equal", bytes(db.profiles.cpu().numpy()) == bytes(pk.profiles),
          "dev inst equal", db.instances.cpu().numpy().tobytes() == pk.instances.tobytes(),
          "inp", np.array_equal(db.inp.cpu().numpy(), pk.inp), "out", np.array_equal(db.out.cpu().numpy(), pk.out))
    db.launch(); s = db.fetch()
    print(name, "status", s["status"][:4], "n", s["n"][:4])
    print(" inst0", pk.instances[0])
    print(" kv", pk.instances["kv_capacity_tokens"][:3], "worst", int((pk.inp.astype(np.int64)+pk.out).max()))
