"""Racecheck probe for the two-lane CpgHinge kernel only (diagnostic)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2502_11129_b200 as hb  # noqa: E402

ex = hb.GpuExecutor(0)
ex.run(hb.BatchRequest(4, np.arange(256, dtype=np.uint64), 30))
