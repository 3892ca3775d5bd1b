"""Deterministic synthetic inputs for the remesh hot path (host-side data preparation).

Restates the SPEC's fixture generator (`gen-fixtures`: primitives plus
defect injection) and the BASELINE.json configs:

  C1  noisy icosphere, subdivision 5 (F=20,480), r <- 1 + 0.01 N(0,1)           seed 1
  C2  40 closed primitives x 5,000 tris = 200,000, interpenetrating, unwelded   seed 2
  C3  100 primitives x 10,000 tris (scale 0.03-0.09, centres in [0.06,0.94]^3)
      + 1% duplicates, 0.5% holes, 0.5% flipped, 50 pokes, trimmed to exactly
      1,000,000                                                                 seed 3
  C4  icosphere subdivision 9 (F=5,242,880) with a 4-term radial displacement   seed 4
  C5  64 meshes, F log-uniform in [5e4, 2e6], recipes C1-C3 cycled              seed 5

Randomness is a counter-based SplitMix64 stream (no numpy Generator / libstdc++
distributions, which differ across versions), so every machine builds identical bytes.
`normalize_unit_cube` restates mesh_io.cpp:393-408 operation for operation.
"""
from __future__ import annotations

import math

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """SplitMix64 outputs for counters offset..offset+n-1 of stream `seed`."""
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
             + (np.arange(offset, offset + n, dtype=np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


class Rng:
    """Sequential draws from one SplitMix64 stream."""

    def __init__(self, seed: int):
        self.seed = seed
        self.ctr = 0

    def u64(self, n: int) -> np.ndarray:
        out = splitmix64(self.seed, n, self.ctr)
        self.ctr += n
        return out

    def uniform(self, n: int) -> np.ndarray:  # [0, 1)
        return (self.u64(n) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)

    def normal(self, n: int) -> np.ndarray:  # Box-Muller
        m = (n + 1) // 2
        u1 = ((self.u64(m) >> np.uint64(11)).astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)
        u2 = self.uniform(m)
        r = np.sqrt(-2.0 * np.log(u1))
        z = np.concatenate([r * np.cos(2 * np.pi * u2), r * np.sin(2 * np.pi * u2)])
        return z[:n]

    def randint(self, lo: int, hi: int, n: int) -> np.ndarray:  # [lo, hi)
        return lo + (self.u64(n) % np.uint64(hi - lo)).astype(np.int64)


# ---------------------------------------------------------------- primitives (closed manifolds)

def icosphere(subdiv: int):
    t = (1.0 + math.sqrt(5.0)) / 2.0
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t], [0, -1, -t],
                  [0, 1, -t], [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4],
                  [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8],
                  [3, 8, 9], [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], np.int64)
    for _ in range(subdiv):
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        key = np.minimum(e[:, 0], e[:, 1]) * (len(v) + 1) + np.maximum(e[:, 0], e[:, 1])
        uniq, inv = np.unique(key, return_inverse=True)
        a = uniq // (len(v) + 1)
        b = uniq % (len(v) + 1)
        mid = v[a] + v[b]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        base = len(v)
        v = np.concatenate([v, mid])
        nf = len(f)
        m01, m12, m20 = (base + inv[:nf], base + inv[nf:2 * nf], base + inv[2 * nf:])
        f = np.concatenate([
            np.stack([f[:, 0], m01, m20], 1), np.stack([f[:, 1], m12, m01], 1),
            np.stack([f[:, 2], m20, m12], 1), np.stack([m01, m12, m20], 1)])
    return v, f.astype(np.int32)


def _grid_faces(nu: int, nv: int, wrap_u: bool, wrap_v: bool, idx) -> np.ndarray:
    faces = []
    for i in range(nu if wrap_u else nu - 1):
        for j in range(nv if wrap_v else nv - 1):
            a, b = idx(i, j), idx((i + 1) % nu, j)
            c, d = idx((i + 1) % nu, (j + 1) % nv), idx(i, (j + 1) % nv)
            faces += [[a, b, c], [a, c, d]]
    return np.array(faces, np.int64)


def torus(nu: int, nv: int, R: float = 1.0, r: float = 0.35):
    u = 2 * np.pi * np.arange(nu) / nu
    w = 2 * np.pi * np.arange(nv) / nv
    U, W = np.meshgrid(u, w, indexing="ij")
    v = np.stack([(R + r * np.cos(W)) * np.cos(U), (R + r * np.cos(W)) * np.sin(U), r * np.sin(W)], -1)
    f = _grid_faces(nu, nv, True, True, lambda i, j: i * nv + j)
    return v.reshape(-1, 3), f.astype(np.int32)


def uv_sphere(nu: int, nl: int, stretch: float = 0.0):
    """nl latitude rings + 2 poles: 2*nu*nl triangles.  stretch>0 makes a capsule."""
    lat = np.pi * (np.arange(nl) + 1) / (nl + 1)
    lon = 2 * np.pi * np.arange(nu) / nu
    L, O = np.meshgrid(lat, lon, indexing="ij")
    z = np.cos(L) + np.sign(np.cos(L)) * stretch
    v = np.stack([np.sin(L) * np.cos(O), np.sin(L) * np.sin(O), z], -1).reshape(-1, 3)
    top, bot = len(v), len(v) + 1
    v = np.concatenate([v, [[0, 0, 1 + stretch], [0, 0, -1 - stretch]]])
    faces = []
    for k in range(nu):
        faces.append([top, k, (k + 1) % nu])
        faces.append([bot, (nl - 1) * nu + (k + 1) % nu, (nl - 1) * nu + k])
    for i in range(nl - 1):
        for k in range(nu):
            a, b = i * nu + k, i * nu + (k + 1) % nu
            c, d = (i + 1) * nu + (k + 1) % nu, (i + 1) * nu + k
            faces += [[a, d, c], [a, c, b]]
    return v, np.array(faces, np.int32)


def cylinder(n: int, m: int, h: float = 2.0):
    """n around, m+1 rings; 2n(m+1) triangles."""
    th = 2 * np.pi * np.arange(n) / n
    zs = np.linspace(-h / 2, h / 2, m + 1)
    Z, T = np.meshgrid(zs, th, indexing="ij")
    v = np.stack([np.cos(T), np.sin(T), Z], -1).reshape(-1, 3)
    top, bot = len(v), len(v) + 1
    v = np.concatenate([v, [[0, 0, h / 2], [0, 0, -h / 2]]])
    faces = []
    for i in range(m):
        for k in range(n):
            a, b = i * n + k, i * n + (k + 1) % n
            c, d = (i + 1) * n + (k + 1) % n, (i + 1) * n + k
            faces += [[a, b, c], [a, c, d]]
    for k in range(n):
        faces.append([top, m * n + k, m * n + (k + 1) % n])
        faces.append([bot, (k + 1) % n, k])
    return v, np.array(faces, np.int32)


def box(k1: int, k2: int, k3: int):
    """Closed box subdivided k1 x k2 x k3; 4(k1k2 + k2k3 + k1k3) triangles."""
    ks = (k1, k2, k3)
    verts = {}
    vlist = []

    def vid(p):
        if p not in verts:
            verts[p] = len(vlist)
            vlist.append(p)
        return verts[p]

    faces = []
    for ax in range(3):
        b, c = (ax + 1) % 3, (ax + 2) % 3
        for side in (0, 1):
            for i in range(ks[b]):
                for j in range(ks[c]):
                    def P(ii, jj):
                        p = [0, 0, 0]
                        p[ax] = side * ks[ax]
                        p[b] = ii
                        p[c] = jj
                        return vid(tuple(p))
                    q = [P(i, j), P(i + 1, j), P(i + 1, j + 1), P(i, j + 1)]
                    if side == 0:
                        q = q[::-1]
                    faces += [[q[0], q[1], q[2]], [q[0], q[2], q[3]]]
    v = np.array(vlist, np.float64) / np.array(ks, np.float64) - 0.5
    v *= np.array(ks, np.float64) / max(ks)
    return v, np.array(faces, np.int32)


def _rotation(rng: Rng) -> np.ndarray:
    q = rng.normal(4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def primitive(kind: int, tris: int):
    if tris == 5000:
        table = [lambda: uv_sphere(50, 50), lambda: torus(50, 50), lambda: box(20, 30, 13),
                 lambda: cylinder(50, 49), lambda: uv_sphere(50, 50, stretch=0.6)]
    elif tris == 10000:
        table = [lambda: uv_sphere(100, 50), lambda: torus(100, 50), lambda: box(20, 30, 38),
                 lambda: cylinder(100, 49), lambda: uv_sphere(100, 50, stretch=0.6)]
    else:
        raise ValueError(tris)
    v, f = table[kind % 5]()
    assert len(f) == tris, (kind, len(f))
    return v, f


def soup(n_prims: int, tris: int, seed: int, scale=(0.06, 0.2), spread=(0.2, 0.8)):
    rng = Rng(seed)
    vs, fs, off = [], [], 0
    for p in range(n_prims):
        v, f = primitive(p, tris)
        R = _rotation(rng)
        s = scale[0] + (scale[1] - scale[0]) * rng.uniform(1)[0]
        c = spread[0] + (spread[1] - spread[0]) * rng.uniform(3)
        vs.append((v @ R.T) * s + c)
        fs.append(f + off)
        off += len(v)
    return np.concatenate(vs), np.concatenate(fs).astype(np.int32)


def inject_defects(v, f, seed: int, dup=0.01, holes=0.005, flipped=0.005, pokes=50):
    """SPEC.md:794 defect injection: duplicate faces, deleted faces (holes), flipped faces,
    random pokes (small flipped tetrahedra pushed through a face)."""
    rng = Rng(seed * 7919 + 1)
    nf = len(f)
    f = f.copy()
    flip_ids = rng.randint(0, nf, int(flipped * nf))
    f[flip_ids] = f[flip_ids][:, ::-1]
    keep = np.ones(nf, bool)
    keep[rng.randint(0, nf, int(holes * nf))] = False
    dup_ids = rng.randint(0, nf, int(dup * nf))
    f = np.concatenate([f[keep], f[dup_ids]])
    vs = [v]
    fs = [f]
    base = len(v)
    for pid in rng.randint(0, len(f), pokes):
        a, b, c = v[f[pid]]
        n = np.cross(b - a, c - a)
        n /= max(np.linalg.norm(n), 1e-300)
        ctr = (a + b + c) / 3.0
        h = 2.0 * np.linalg.norm(b - a)
        tip_out, tip_in = ctr + h * n, ctr - h * n
        vs.append(np.stack([a, b, c, tip_out, tip_in]))
        i = base
        fs.append(np.array([[i, i + 1, i + 3], [i + 1, i + 2, i + 3], [i + 2, i, i + 3],
                            [i + 1, i, i + 4], [i + 2, i + 1, i + 4], [i, i + 2, i + 4]], np.int64))
        base += 5
    return np.concatenate(vs), np.concatenate(fs).astype(np.int32)


def nested_shells(subdiv: int, gap: float, k: int, seed: int):
    """k concentric noisy icospheres 1 + i*gap apart (alternating orientation): a thin-wall
    fixture on which collapses poke through the neighbouring wall, so undo loops
    need 2-3 rounds."""
    v, f = icosphere(subdiv)
    rng = Rng(seed)
    n = len(v)
    vs, fs = [], []
    for i in range(k):
        vs.append(v * (1.0 + i * gap + 0.1 * gap * rng.normal(n))[:, None])
        fs.append((f[:, ::-1] if i % 2 == 0 else f) + i * n)
    return np.concatenate(vs), np.concatenate(fs).astype(np.int32)


def normalize_unit_cube(v: np.ndarray, padding: float):
    """mesh_io.cpp:393-408: uniform scale into [padding, 1-padding]^3, centred."""
    if not (0 <= padding < 0.5):
        raise ValueError("normalize_unit_cube: padding must be in [0, 0.5)")
    lo = v.min(axis=0)
    hi = v.max(axis=0)
    ext = hi - lo
    longest = float(max(ext[0], ext[1], ext[2]))
    if not longest > 0:
        raise ValueError("normalize_unit_cube: all vertices coincide")
    scale = (1.0 - 2.0 * padding) / longest
    center = (lo + hi) * 0.5
    translation = 0.5 - center * scale
    return v * scale + translation, (scale, translation)


# ---------------------------------------------------------------- BASELINE configs

CONFIGS = {
    "c1": dict(R=128, target=5000),
    "c2": dict(R=256, target=20000),
    "c3": dict(R=512, target=50000),
    "c4": dict(R=1024, target=None),
}


def make_config(name: str):
    """Returns (vertices normalised with padding 6/R, faces, R, target)."""
    name = name.lower()
    cfg = CONFIGS[name]
    R = cfg["R"]
    if name == "c1":
        v, f = icosphere(5)
        r = 1.0 + 0.01 * Rng(1).normal(len(v))
        v = v * r[:, None]
    elif name == "c2":
        v, f = soup(40, 5000, seed=2)
    elif name == "c3":
        # primitive scale/spread chosen so the remeshed soup keeps few enclosed pockets: the
        # 50k-face target is then above the topological floor of the DMC output (a denser
        # arrangement seals ~20k pockets whose minimal meshes alone exceed 50k faces)
        v, f = soup(100, 10000, seed=3, scale=(0.03, 0.09), spread=(0.06, 0.94))
        v, f = inject_defects(v, f, seed=3)
        f = f[:1_000_000]
        used = np.zeros(len(v), bool)
        used[f.ravel()] = True
        remap = np.cumsum(used) - 1
        v, f = v[used], remap[f].astype(np.int32)
    elif name == "c4":
        v, f = icosphere(9)
        rng = Rng(4)
        k = rng.normal(12).reshape(4, 3)
        amp = 0.02 * rng.uniform(4)
        r = 1.0 + sum(amp[i] * np.sin(v @ k[i] * 3.0) for i in range(4))
        v = v * r[:, None]
    else:
        raise ValueError(name)
    v, _ = normalize_unit_cube(np.ascontiguousarray(v, np.float64), 6.0 / R)
    return np.ascontiguousarray(v), np.ascontiguousarray(f, np.int32), R, cfg["target"]


def add_bowties(v, f, seed: int, n: int):
    """Bowtie (non-manifold) vertices: n random vertex pairs from different parts of
    the soup are merged into one index."""
    rng = Rng(seed * 104729 + 7)
    f = f.copy()
    a = rng.randint(0, len(v), n)
    b = rng.randint(0, len(v), n)
    for i, j in zip(a.tolist(), b.tolist()):
        if i != j:
            f[f == j] = i
    keep = (f[:, 0] != f[:, 1]) & (f[:, 1] != f[:, 2]) & (f[:, 0] != f[:, 2])  # load_mesh drops these
    return v, f[keep]


def defect_corpus(n: int = 20, seed: int = 6):
    """SPEC.md:805 acceptance #1 corpus: n fixtures with 5k-300k input faces (log-spaced), soups of
    interpenetrating primitives with duplicate faces, holes, flipped faces, poked tetrahedra and
    bowtie vertices.  Returns [(raw vertices, faces, R, target)] with R alternating 64 / 128 and a
    1% face target."""
    out = []
    for i in range(n):
        F = int(round(math.exp(math.log(5e3) + (math.log(3e5) - math.log(5e3)) * i / max(n - 1, 1))))
        per = 5000 if F < 200000 else 10000
        v, f = soup(max(1, F // per), per, seed=seed * 1000 + i, scale=(0.1, 0.35), spread=(0.25, 0.75))
        v, f = inject_defects(v, f, seed=seed * 1000 + i, pokes=5 + i)
        v, f = add_bowties(v, f, seed * 1000 + i, 3)
        R = 64 if i % 2 == 0 else 128
        out.append((np.ascontiguousarray(v * 2.0 - 0.3), np.ascontiguousarray(f, np.int32), R, max(4, len(f) // 100)))
    return out


def c5_batch(n: int = 64, seed: int = 5):
    """C5: n meshes, F log-uniform in [5e4, 2e6], recipes C1-C3 cycled (resolution by the SPEC
    auto rule: target = 1% of F -> R = 128 if target < 1000 else 256)."""
    rng = Rng(seed)
    out = []
    for i in range(n):
        F = int(round(math.exp(math.log(5e4) + (math.log(2e6) - math.log(5e4)) * rng.uniform(1)[0])))
        target = max(4, F // 100)
        R = 128 if target < 1000 else 256
        kind = i % 3
        if kind == 0:
            sub = max(1, int(round(math.log(F / 20) / math.log(4))))
            v, f = icosphere(sub)
            v = v * (1.0 + 0.01 * Rng(1000 + i).normal(len(v)))[:, None]
        else:
            per = 5000 if F < 400000 else 10000
            v, f = soup(max(1, F // per), per, seed=1000 + i)
            if kind == 2:
                v, f = inject_defects(v, f, seed=1000 + i, pokes=5)
        v, _ = normalize_unit_cube(v, 6.0 / R)
        out.append((np.ascontiguousarray(v), np.ascontiguousarray(f, np.int32), R, target))
    return out
