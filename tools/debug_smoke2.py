import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_02329_b200.batch import config1, run_batch
from paper_2605_02329_b200.engine import run_packed
sw = config1(); got = run_batch(sw.packed).copy()
print("device path:", got[0])
sw2 = config1(); run_packed(sw2.packed); print("host path:", sw2.packed.summaries[0])
