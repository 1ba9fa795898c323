"""Emulate the table-driven exp64 of contract.cuh in numpy (fp64) and report its max relative
error against numpy's exp over the compositing range and the full valid range."""
import math

import numpy as np

L = math.log(2) / 256
for lo in (-6.0, -700.0):
    x = np.linspace(lo, 0.0, 4_000_001)
    k = np.rint(x / L)
    r = x - k * L
    p = 1 + r * (1 + r * (0.5 + r / 6))
    v = np.exp2(np.mod(k, 256) / 256) * p * np.exp2(np.floor(k / 256))
    print(f"[{lo}, 0]: max relative error {np.max(np.abs(v / np.exp(x) - 1)):.2e}")
