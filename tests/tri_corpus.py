"""Generated triangle-pair corpus (coplanar, sharp, vertex-sharing and
edge-sharing cases).  Deterministic (SplitMix64)."""
import numpy as np

from paper_2509_05595_b200.fixtures import Rng


def corpus(n: int, seed: int = 0):
    """Returns (vertices, faces, pairs) with n pairs spread over the case families."""
    rng = Rng(seed)
    verts, faces, pairs = [], [], []

    def add_tri(p):
        base = len(verts)
        verts.extend(p)
        faces.append([base, base + 1, base + 2])
        return len(faces) - 1

    def rnd(k):
        return rng.uniform(3 * k).reshape(k, 3)

    grid = lambda k: np.round(rng.uniform(3 * k).reshape(k, 3) * 4) / 4  # snapped: many exact cases
    for i in range(n):
        kind = i % 8
        if kind == 0:    # random
            t1, t2 = rnd(3), rnd(3)
        elif kind == 1:  # snapped to a coarse lattice (exact coplanar / touching cases)
            t1, t2 = grid(3), grid(3)
        elif kind == 2:  # coplanar z=0.5
            t1, t2 = rnd(3), rnd(3)
            t1[:, 2] = 0.5
            t2[:, 2] = 0.5
        elif kind == 3:  # sharp: nearly parallel
            t1 = rnd(3)
            t2 = t1 + 1e-9 * (rnd(3) - 0.5)
            t2 = t2[[1, 2, 0]]
        elif kind in (4, 5):  # shared vertex (index) — kind 5 coplanar
            t1 = rnd(3)
            t2 = rnd(3)
            if kind == 5:
                t1[:, 2] = 0.25
                t2[:, 2] = 0.25
            base = len(verts)
            verts.extend(t1)
            verts.extend(t2[1:])
            faces.append([base, base + 1, base + 2])
            faces.append([base, base + 3, base + 4])
            pairs.append([len(faces) - 2, len(faces) - 1])
            continue
        else:            # shared edge — kind 7 coplanar
            t1 = rnd(3)
            d = rnd(1)
            if kind == 7:
                t1[:, 2] = 0.75
                d[:, 2] = 0.75
            base = len(verts)
            verts.extend(t1)
            verts.extend(d)
            faces.append([base, base + 1, base + 2])
            faces.append([base + 1, base, base + 3])
            pairs.append([len(faces) - 2, len(faces) - 1])
            continue
        a = add_tri(list(t1))
        b = add_tri(list(t2))
        pairs.append([a, b])
    return np.array(verts, np.float64), np.array(faces, np.int32), np.array(pairs, np.int32)
