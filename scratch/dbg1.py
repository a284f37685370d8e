import sys, numpy as np
sys.path.insert(0, '.')
from paper_2209_04579_b200 import tqp
rng = np.random.default_rng(0)
for n in (100, 2048, 2049, 5000, 30000, 300000):
    x = rng.integers(0, 2, n).astype(np.int64)
    got = tqp.prefix_sum_exclusive(x.reshape(-1,1)).numpy().ravel()
    want = np.concatenate([[0], np.cumsum(x)[:-1]])
    bad = np.flatnonzero(got != want)
    print(n, "prefix ok" if bad.size == 0 else f"prefix BAD first={bad[:5]} got={got[bad[:5]]} want={want[bad[:5]]}")
    m = (rng.random(n) < 0.5).astype(np.uint8)
    idx = tqp.compact(np.arange(n, dtype=np.int64).reshape(-1,1), m.reshape(-1,1)).numpy().ravel()
    print(n, "compact ok" if np.array_equal(idx, np.flatnonzero(m)) else "compact BAD")
    k = rng.integers(0, 5, n).astype(np.int64)
    p = tqp.argsort_stable(k.reshape(-1,1)).numpy().ravel()
    print(n, "argsort ok" if np.array_equal(p, np.argsort(k, kind='stable')) else "argsort BAD")
