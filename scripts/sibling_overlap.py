"""Developer analysis: how many far-list entries siblings share (t far from both
children of one parent) -- the atomics a sibling-merged M2T would save."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2106_04487_b200 as fkt

C = {2: ("matern32", {"sigma": 1.0, "rho": 0.1}, 1000000, 6, 512, 0.5),
     4: ("inverse-r", {}, 4000000, 8, 512, 0.5),
     5: ("cauchy", {"sigma": 1.0}, 2000000, 6, 512, 0.75)}
for cfg in [int(a) for a in sys.argv[1:]] or [5]:
    name, prm, n, p, leaf, theta = C[cfg]
    x, w = fkt.synthConfig(cfg, n)
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, prm), fkt.FktOptions(p=p, theta=theta, leafCapacity=leaf))
    t = pl.tree()
    fo, fi = t.farCsr()
    tot = int(fo[-1]); shared = 0
    for b in range(t.nodeCount()):
        l, r = int(t.lefts[b]), int(t.rights[b])
        if l < 0 or r < 0:
            continue
        a = fi[fo[l]:fo[l + 1]]; c = fi[fo[r]:fo[r + 1]]
        shared += np.intersect1d(a, c, assume_unique=True).size
    print(f"cfg{cfg}: far entries {tot}, entries shared by siblings {2 * shared} ({200.0 * shared / tot:.1f}%), "
          f"atomics saved by sibling merging {shared} ({100.0 * shared / tot:.1f}%)")
