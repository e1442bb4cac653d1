"""Compare two tools/ab_dump.py outputs field by field: python tools/ab_cmp.py A.npz B.npz"""
import sys

import numpy as np

a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
print("identical" if not bad else f"DIFFER: {bad}")
