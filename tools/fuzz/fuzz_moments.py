"""Random design matrices through K1 (compute_scatter): band counts 1-32, 2-40 classes
(several moment launches), 50-400k points (one chunk per CTA, two chunks, the 1024-CTA cap),
sorted and shuffled labels, against the oracle's two-pass scatter
(dev tool; python tools/fuzz/fuzz_moments.py [seed])."""
import sys, traceback
ROOT = __import__('pathlib').Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / 'tests'))
import numpy as np
import oracle
from golden_util import rel_close
import paper_1612_06457_b200 as ut
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
fails = 0
for it in range(120):
    try:
        b = int(rng.integers(1, 33)); c = int(rng.integers(2, 41))
        n = int(rng.choice([rng.integers(c, 300), rng.integers(300, 40000), rng.integers(40000, 400000)]))
        labels = rng.integers(0, c, n); labels[:c] = np.arange(c)
        if it % 3 == 0:
            labels = np.sort(labels)
        offs = rng.uniform(-5, 5, size=(b, 1)) * (10.0 ** rng.integers(-2, 4))
        values = offs + rng.normal(size=(b, n)) * rng.uniform(0.01, 2.0, size=(b, 1)) + 0.1 * labels[None, :]
        sp = ut.compute_scatter(ut.DesignMatrix(np.ascontiguousarray(values), labels.astype(np.intp), tuple()))
        want = oracle.scatter(values, labels)
        case = (b, c, n, it % 3 == 0)
        assert np.array_equal(sp.counts, want["counts"]), ("counts",) + case
        for got, key in ((sp.within, "within"), (sp.between, "between"),
                         (sp.class_means, "class_means"), (sp.grand_mean, "grand_mean")):
            assert rel_close(got, want[key], 1e-9), (key,) + case
    except Exception as e:
        fails += 1
        print("FAIL", it, repr(e)[:200], traceback.format_exc().splitlines()[-3][:140], flush=True)
print("fuzz moments done, fails:", fails)
