"""Quick GPU parity of the default plan at a few sizes (for A/B builds via BW_LIB_PATH)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1607_01039_b200 as bw  # noqa: E402
from oracle import load_c, oracle_np  # noqa: E402

lib = load_c()
ok = True
for n in (22, 23, 24, 26):
    x = oracle_np.gen(2, n, [1 << 20], 0, 1 << n)
    t = torch.from_numpy(x).cuda()
    bw.fwht_array(t)
    r = x.copy()
    lib.oracle_fwht_i64(r.ctypes.data, n)
    good = np.array_equal(t.cpu().numpy(), r)
    ok &= good
    print("parity", n, good)
print("ALL OK" if ok else "MISMATCH")
