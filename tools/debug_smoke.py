import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle
from paper_2605_02329_b200.batch import config1, run_batch
sw = config1(); got = run_batch(sw.packed).copy()
ref = config1(synth=oracle.synth); oracle.run_batch(ref.packed, threads=4); want = ref.packed.summaries
for k in want.dtype.names:
    if not np.array_equal(got[k], want[k], equal_nan=(got[k].dtype.kind=='f')):
        print(k, "gpu", got[k].tolist(), "\n   oracle", want[k].tolist())
