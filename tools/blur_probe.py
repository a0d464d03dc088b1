"""Probe the 3D blur on one (shape, R): bit-exact vs the oracle's device order.
    python tools/blur_probe.py nx ny nz R"""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1308_6634_b200 as mb
import pyoracle
nx, ny, nz, R = map(int, sys.argv[1:5])
orc = pyoracle.Oracle()
orc.set_device_order(1)
shape = (nx, ny, nz)
taps = orc.taps(nx, 0.05, radius=R)
x = np.random.default_rng(1).uniform(-1, 1, nx * ny * nz)
y = mb.SeparableGaussianBlur(shape, taps=taps).apply(x)
ref = orc.blur(3, shape, taps).apply(x)
print(shape, R, "bit-exact" if np.array_equal(y, ref) else f"MISMATCH max {np.abs(y - ref).max()}")
