"""Seeded activation schedule of the calibration-statistics fixture (shared by
make_calib.py, which feeds it to the reference, and tests/test_calibration.py)."""
import numpy as np

# (site, shape, scale): values ~ standard_t(3) * scale, float32.  layers.0.x totals
# 4.5M values > POOL_CAP (2^22), so the seeded reservoir runs.
STATS_PLAN = [("layers.0.in", (300, 64), 1.0), ("layers.0.x", (1500, 1000), 0.3), ("layers.0.b", (700, 16), 2.0),
              ("layers.0.x", (1400, 1000), 0.5), ("layers.0.dt", (4, 3), 0.01), ("layers.0.x", (1600, 1000), 0.2),
              ("layers.0.b", (5, 16), 9.0), ("layers.0.y", (2, 8), 0.0)]


def stats_activations(seed=123):
    rng = np.random.default_rng(seed)
    return [(site, (rng.standard_t(3, size=shape) * s).astype(np.float32)) for site, shape, s in STATS_PLAN]
