"""C4-size dense operator driver for ncu: python tools/c4_driver.py (64^3 voxels x 4096 rows)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1308_6634_b200 as mb  # noqa: E402

op = mb.FdotOperator(64, 64, 64, seed=4)
x = torch.rand(64 ** 3, dtype=torch.float64, device="cuda")
y = torch.rand(4096, dtype=torch.float64, device="cuda")
for _ in range(3):
    a = op.apply(x)
    b = op.apply_adjoint(y)
torch.cuda.synchronize()
