import sys, os, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2605_02329_b200.batch import config5, run_batch
s = run_batch(config5(select=np.array([130145])).packed)
print(s[0][['decode_steps','digest']])
