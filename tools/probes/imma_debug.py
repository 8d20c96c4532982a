"""Debug probe for the integer region-moments path: prints device vs numpy
moments for small structured cubes."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests")
from test_gpu_region import moments, reference  # noqa: E402

np.set_printoptions(precision=6, linewidth=150)


def show(name, cube):
    n, mean, m2 = moments(cube)
    rn, rmean, rm2 = reference(cube)
    print(f"== {name} n={n} ref_n={rn}")
    print(" mean", mean, "ref", rmean, "dsum", (mean - rmean) * n)
    print(" m2 diag", np.diag(m2), "ref", np.diag(rm2))


c = np.full((1, 16, 256), 100, np.uint8)
show("const100", c)
c2 = c.copy(); c2[0, 0, 0] = 101
show("one+1 at px0", c2)
c3 = c.copy(); c3[0, 0, 5] = 102
show("one+2 at px5", c3)
c4 = c.copy(); c4[0, 3, 17] = 90
show("one-10 at px 785", c4)
c5 = np.full((1, 1, 512), 100, np.uint8); c5[0, 0, 300] = 110
show("512px +10 at 300", c5)
c6 = np.full((2, 16, 256), 100, np.uint8); c6[1] = 50; c6[1, 0, 1] = 52
show("2 bands", c6)
rng = np.random.default_rng(0)
c7 = rng.integers(90, 110, size=(1, 16, 256)).astype(np.uint8)
show("random 1 band 4096", c7)
c8 = rng.integers(90, 110, size=(1, 40, 100)).astype(np.uint8)
show("random 1 band 4000", c8)
