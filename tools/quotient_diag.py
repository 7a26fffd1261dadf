import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import test_gpu_quotients as t
for name, op in sorted(t.OPS.items()):
    rng = np.random.default_rng(op + 100)
    n = 1 << 20
    d = t.DIVISORS[name](rng, n)
    for cls, x in t.numerators(rng, n).items():
        got = t.run(op, x, d); want = x / d
        bad = ~t.same(got, want)
        if bad.any():
            i = np.flatnonzero(bad)[:2]
            print(name, cls, int(bad.sum()), [(float(x[k]), float(d[k]), float(got[k]), float(want[k])) for k in i])
        else:
            print(name, cls, "ok")
