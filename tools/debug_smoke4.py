import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_02329_b200.batch import config1, config3, DeviceBatch
from paper_2605_02329_b200 import _abi
L = _abi.lib()
a = config1().packed
db = DeviceBatch(a)
for k in range(3):
    db.summaries.zero_(); db.launch(); s = db.fetch(); print("config1 launch", k, s["status"][:6], flush=True)
c3 = config3(select=np.arange(0, 3072, 7)).packed
db3 = DeviceBatch(c3)
for k in range(2):
    db3.summaries.zero_(); db3.launch(); s = db3.fetch(); print("config3 launch", k, np.unique(s["status"]), flush=True)
for k in range(2):
    db.summaries.zero_(); db.launch(); s = db.fetch(); print("config1 again", k, s["status"][:6], flush=True)
