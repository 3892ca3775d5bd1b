"""CPU restatement of one stage-3 Newton step — TEST INFRASTRUCTURE ONLY.

Only tests/ may import this module (the step oracle of tests/test_gpu_project_steps.py).  It
restates SPEC.md's safe_project energies in float64 with
torch's CPU autograd for the derivatives, so nothing here shares code with the GPU's forward-mode
jets (csrc/project.cu):

  rest_state      X0 -> per-face Dm^-1 and A0 (2D frames), barycentric vertex
                  areas s0, interior hinges with rest dihedral / edge length
                  
  pt_class /      frozen distance classes: point-vertex, point-edge, point-plane;
  ee_class        edge-edge: vertex-vertex, vertex-edge, line-line
  energy          B(X) = k_dis (E_S2M + E_M2S) + k_elas E_elas + k_bend E_bend + k_bar sum b(d)
                  with the targets, classes and contact set frozen
  gradient        autograd of `energy`
  hessian_spd     per-stencil autograd Hessians, eigenvalues < 1e-10 clamped,
                  assembled into a scipy CSR matrix
  contacts        brute-force contact set: every point-triangle / edge-edge pair that shares no
                  vertex with d < d̂
  accd            additive CCD over the swept primitive pairs (slack 0.9,
                  margin 0.1 d̂, at most 64 advancements per pair)

Parity is pinned to SPEC's formulas and to the GPU trace (targets, classes and contacts are
checked separately before they are used).  The reference ships no safe_project source
(SURVEY.md §2 row 13), so there is no reference output to pin against: parity unpinned beyond
SPEC.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import torch

PT, EE = 4, 5
LAMBDA_FLOOR = 1e-10


# ------------------------------------------------------------------------------ rest state
def rest_state(X0: np.ndarray, F: np.ndarray) -> dict:
    x0, x1, x2 = X0[F[:, 0]], X0[F[:, 1]], X0[F[:, 2]]
    e1, e2 = x1 - x0, x2 - x0
    n = np.cross(e1, e2)
    nl = np.linalg.norm(n, axis=1)
    l1 = np.linalg.norm(e1, axis=1)
    if not (np.all(l1 > 0) and np.all(nl > 0)):
        raise ValueError("degenerate rest face")
    u = e1 / l1[:, None]
    w = np.cross(n / nl[:, None], u)
    # Dm = [[e1.u, e2.u], [e1.w, e2.w]] = [[l1, e2.u], [0, e2.w]]
    m00, m01, m11 = l1, np.einsum("ij,ij->i", e2, u), np.einsum("ij,ij->i", e2, w)
    dminv = np.zeros((len(F), 2, 2))
    dminv[:, 0, 0] = 1.0 / m00
    dminv[:, 0, 1] = -m01 / (m00 * m11)
    dminv[:, 1, 1] = 1.0 / m11
    a0 = 0.5 * nl
    s0 = np.zeros(len(X0))
    for k in range(3):
        np.add.at(s0, F[:, k], a0 / 3.0)
    # interior edges -> hinges (i, j | k, l): faces (i, j, k) and (j, i, l)
    he = {}
    for f, tri in enumerate(F):
        for k in range(3):
            a, b = int(tri[k]), int(tri[(k + 1) % 3])
            he.setdefault((min(a, b), max(a, b)), []).append((a, b, int(tri[(k + 2) % 3])))
    hinges = []
    for lst in he.values():
        if len(lst) == 2:
            (a, b, c), (_, _, d) = lst
            hinges.append((a, b, c, d))
    hinges = np.array(hinges, np.int64).reshape(-1, 4)
    th0 = dihedral(torch.from_numpy(X0[hinges])).numpy() if len(hinges) else np.zeros(0)
    l0 = np.linalg.norm(X0[hinges[:, 1]] - X0[hinges[:, 0]], axis=1)
    edges = np.array(sorted(he.keys()), np.int64).reshape(-1, 2)
    return {"dminv": dminv, "a0": a0, "s0": s0, "hinges": hinges, "theta0": th0, "l0": l0, "edges": edges}


def dihedral(x):  # x: (..., 4, 3) hinge (i, j, k, l); signed, flat = 0
    e = x[..., 1, :] - x[..., 0, :]
    n0 = torch.linalg.cross(e, x[..., 2, :] - x[..., 0, :])
    n1 = torch.linalg.cross(x[..., 3, :] - x[..., 0, :], e)
    el = torch.sqrt((e * e).sum(-1))
    sn = (torch.linalg.cross(n0, n1) * e).sum(-1) / el
    return torch.atan2(sn, (n0 * n1).sum(-1))


# -------------------------------------------------------------------------- distance classes
def pt_class(p, t0, t1, t2) -> np.ndarray:
    """0..2 nearest vertex t_k, 3..5 edge (t0t1, t1t2, t2t0), 6 interior of the plane."""
    p, t0, t1, t2 = (np.atleast_2d(a) for a in (p, t0, t1, t2))
    e0, e1, w = t1 - t0, t2 - t0, p - t0
    n = np.cross(e0, e1)
    nn = (n * n).sum(1)
    d00, d01, d11 = (e0 * e0).sum(1), (e0 * e1).sum(1), (e1 * e1).sum(1)
    d20, d21 = (w * e0).sum(1), (w * e1).sum(1)
    with np.errstate(divide="ignore", invalid="ignore"):
        den = d00 * d11 - d01 * d01
        bv = (d11 * d20 - d01 * d21) / den
        bw = (d00 * d21 - d01 * d20) / den
    inside = (nn > 0) & (bv > 0) & (bw > 0) & (bv + bw < 1)
    T = (t0, t1, t2)
    best = np.full(len(p), np.inf)
    cls = np.zeros(len(p), np.int64)
    for e in range(3):
        a, b = T[e], T[(e + 1) % 3]
        ab, ap = b - a, p - a
        den = (ab * ab).sum(1)
        with np.errstate(divide="ignore", invalid="ignore"):
            t = np.where(den > 0, (ap * ab).sum(1) / den, 0.0)
        t = np.clip(t, 0.0, 1.0)
        q = ap - t[:, None] * ab
        d2 = (q * q).sum(1)
        c = np.where(t <= 0, e, np.where(t >= 1, (e + 1) % 3, 3 + e))
        better = d2 < best
        best = np.where(better, d2, best)
        cls = np.where(better, c, cls)
    return np.where(inside, 6, cls)


def ee_class(a0, a1, b0, b1) -> np.ndarray:
    """0..3 endpoint pairs (a0b0, a0b1, a1b0, a1b1), 4..7 endpoint-segment (a0-b, a1-b, b0-a,
    b1-a), 8 interior-interior."""
    a0, a1, b0, b1 = (np.atleast_2d(x) for x in (a0, a1, b0, b1))
    u, v, w = a1 - a0, b1 - b0, a0 - b0
    a, b, c = (u * u).sum(1), (u * v).sum(1), (v * v).sum(1)
    d, e = (u * w).sum(1), (v * w).sum(1)
    D = a * c - b * b
    with np.errstate(divide="ignore", invalid="ignore"):
        s, t = (b * e - c * d) / D, (a * e - b * d) / D
    interior = (D > 1e-12 * a * c) & (s > 0) & (s < 1) & (t > 0) & (t < 1)
    P, S0, S1 = (a0, a1, b0, b1), (b0, b0, a0, a0), (b1, b1, a1, a1)
    best = np.full(len(a0), np.inf)
    cls = np.zeros(len(a0), np.int64)
    for q in range(4):
        sv, spv = S1[q] - S0[q], P[q] - S0[q]
        den = (sv * sv).sum(1)
        with np.errstate(divide="ignore", invalid="ignore"):
            tt = np.where(den > 0, (spv * sv).sum(1) / den, 0.0)
        tt = np.clip(tt, 0.0, 1.0)
        r = spv - tt[:, None] * sv
        d2 = (r * r).sum(1)
        if q < 2:
            c_end = (0 if q == 0 else 2) + (tt >= 1)
        else:
            c_end = 2 * (tt >= 1) + (0 if q == 2 else 1)
        c = np.where((tt > 0) & (tt < 1), 4 + q, c_end)
        better = d2 < best
        best = np.where(better, d2, best)
        cls = np.where(better, c, cls)
    return np.where(interior, 8, cls)


def _pp(a, b):
    d = a - b
    return (d * d).sum(-1)


def _pe(p, a, b):
    c = torch.linalg.cross(a - p, b - p)
    e = b - a
    return (c * c).sum(-1) / (e * e).sum(-1)


def _plane(p, t0, t1, t2):
    n = torch.linalg.cross(t1 - t0, t2 - t0)
    s = ((p - t0) * n).sum(-1)
    return s * s / (n * n).sum(-1)


def d2_pt(p, t, cls: int):  # t: (..., 3, 3)
    if cls < 3:
        return _pp(p, t[..., cls, :])
    if cls < 6:
        return _pe(p, t[..., cls - 3, :], t[..., (cls - 2) % 3, :])
    return _plane(p, t[..., 0, :], t[..., 1, :], t[..., 2, :])


def d2_ee(x, cls: int):  # x: (..., 4, 3) = a0, a1, b0, b1
    a0, a1, b0, b1 = x[..., 0, :], x[..., 1, :], x[..., 2, :], x[..., 3, :]
    if cls < 4:
        return _pp((a0, a0, a1, a1)[cls], (b0, b1, b0, b1)[cls])
    if cls < 8:
        p, s0, s1 = ((a0, b0, b1), (a1, b0, b1), (b0, a0, a1), (b1, a0, a1))[cls - 4]
        return _pe(p, s0, s1)
    n = torch.linalg.cross(a1 - a0, b1 - b0)
    s = ((b0 - a0) * n).sum(-1)
    return s * s / (n * n).sum(-1)


# ------------------------------------------------------------------------------- the energy
class StepOracle:
    """B(X) with frozen data: targets (nv x 3), M2S stencils (m x 4: face vertices + class),
    samples (m x 3), contacts (c x 6: term, class, 4 vertices)."""

    def __init__(self, X0, F, Vin, Fin, params: dict):
        self.F = np.asarray(F, np.int64)
        self.P = params
        self.rest = rest_state(np.asarray(X0, np.float64), self.F)
        self.nv = len(X0)
        a = 0.5 * np.linalg.norm(np.cross(Vin[Fin[:, 1]] - Vin[Fin[:, 0]], Vin[Fin[:, 2]] - Vin[Fin[:, 0]]), axis=1)
        self.m2s_w = float(a.sum()) / float(params["samples"])
        self.t = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in self.rest.items()}

    # -- per-term stencil energies: x is (S, k, 3) for S stencils of k vertices
    def _elastic(self, x, faces):
        P = self.P
        e1, e2 = x[:, 1] - x[:, 0], x[:, 2] - x[:, 0]
        mi = self.t["dminv"][faces]
        f1 = mi[:, 0, 0, None] * e1 + mi[:, 1, 0, None] * e2
        f2 = mi[:, 0, 1, None] * e1 + mi[:, 1, 1, None] * e2
        c11, c22, c12 = (f1 * f1).sum(-1) - 1.0, (f2 * f2).sum(-1) - 1.0, (f1 * f2).sum(-1)
        s = c11 * c11 + c22 * c22 + 2.0 * c12 * c12
        w = 0.25 * self.t["a0"][faces] * P["kelas"]
        if int(P["elas_power"]) == 2:
            return w * s
        tau = P["elas_tau"]
        lo = s.detach() < tau
        blend = s * (3.0 * tau - s) * (0.5 / (tau * np.sqrt(tau)))
        root = torch.sqrt(torch.where(lo, torch.ones_like(s), s))
        return w * torch.where(lo, blend, root)

    def _bend(self, x, hinges):
        dth = dihedral(x) - self.t["theta0"][hinges]
        return 0.5 * self.P["kbend"] * self.t["l0"][hinges] * dth * dth

    def _barrier(self, d2):
        dhat = self.P["dhat"]
        d = torch.sqrt(d2)
        return self.P["kbar"] * (-(d - dhat) ** 2 * torch.log(d / dhat))

    def stencils(self, targets, m2s, samples, contacts):
        """[(kind, vertex index array (S, k), energy function of (S, k, 3))] for every group of
        stencils that shares one closed form."""
        P = self.P
        out = []
        s0 = self.t["s0"]
        tg = torch.from_numpy(np.ascontiguousarray(targets))
        vid = np.arange(self.nv)[:, None]
        out.append(("s2m", vid, lambda x, ix=vid: P["kdis"] * s0[ix[:, 0]] * _pp(x[:, 0], tg[ix[:, 0]])))
        ys = torch.from_numpy(np.ascontiguousarray(samples))
        m2s = np.asarray(m2s)
        for c in range(7):
            sel = np.nonzero(m2s[:, 3] == c)[0]
            if len(sel):
                out.append(("m2s", m2s[sel, :3].astype(np.int64),
                            lambda x, c=c, sel=sel: (P["kdis"] * self.m2s_w) * d2_pt(ys[sel], x, c)))
        faces = np.arange(len(self.F))
        out.append(("elastic", self.F, lambda x: self._elastic(x, faces)))
        hs = np.arange(len(self.rest["hinges"]))
        if len(hs):
            out.append(("bend", self.rest["hinges"], lambda x: self._bend(x, hs)))
        contacts = np.asarray(contacts).reshape(-1, 6)
        for term in (PT, EE):
            for c in range(9):
                sel = np.nonzero((contacts[:, 0] == term) & (contacts[:, 1] == c))[0]
                if len(sel) == 0:
                    continue
                if term == PT:
                    fn = lambda x, c=c: self._barrier(d2_pt(x[:, 0], x[:, 1:4], c))
                else:
                    fn = lambda x, c=c: self._barrier(d2_ee(x, c))
                out.append(("pt" if term == PT else "ee", contacts[sel, 2:6].astype(np.int64), fn))
        return out

    def energy_grad(self, X, targets, m2s, samples, contacts):
        Xt = torch.tensor(np.asarray(X, np.float64), requires_grad=True)
        parts = {}
        for kind, ix, fn in self.stencils(targets, m2s, samples, contacts):
            v = fn(Xt[torch.from_numpy(ix)]).sum()
            parts[kind] = parts.get(kind, 0.0) + v
        B = sum(parts.values())
        (g,) = torch.autograd.grad(B, Xt)
        return float(B.detach()), g.numpy().copy(), {k: float(v.detach()) for k, v in parts.items()}

    def energy(self, X, targets, m2s, samples, contacts) -> float:
        with torch.no_grad():
            Xt = torch.from_numpy(np.asarray(X, np.float64))
            return float(sum(fn(Xt[torch.from_numpy(ix)]).sum()
                             for _, ix, fn in self.stencils(targets, m2s, samples, contacts)))

    def hessian_spd(self, X, targets, m2s, samples, contacts) -> sp.csr_matrix:
        """Per-stencil autograd Hessians, SPD-clamped (eigenvalues < 1e-10 -> 1e-10), summed."""
        Xt = torch.from_numpy(np.asarray(X, np.float64))
        rows, cols, vals = [], [], []
        for _, ix, fn in self.stencils(targets, m2s, samples, contacts):
            S, k = ix.shape
            x = Xt[torch.from_numpy(ix)].reshape(S, 3 * k).clone().requires_grad_(True)
            e = fn(x.reshape(S, k, 3)).sum()
            (g,) = torch.autograd.grad(e, x, create_graph=True)
            H = torch.zeros(S, 3 * k, 3 * k, dtype=torch.float64)
            for j in range(3 * k):  # stencils are independent: d(sum g[:, j]) / dx gives row j of each block
                (hj,) = torch.autograd.grad(g[:, j].sum(), x, retain_graph=True)
                H[:, j, :] = hj
            H = 0.5 * (H + H.transpose(1, 2))
            lam, Q = torch.linalg.eigh(H)
            lam = torch.clamp(lam, min=LAMBDA_FLOOR)
            H = (Q * lam[:, None, :]) @ Q.transpose(1, 2)
            dof = (3 * ix[:, :, None] + np.arange(3)).reshape(S, 3 * k)
            rows.append(np.repeat(dof, 3 * k, axis=1).ravel())
            cols.append(np.tile(dof, (1, 3 * k)).ravel())
            vals.append(H.detach().numpy().ravel())
        n = 3 * self.nv
        return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsr()


# --------------------------------------------------------------------------------- contacts
def _edge_ids(F):
    e = np.sort(np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]]), axis=1)
    return np.unique(e, axis=0)


def pt_distance2(X, pv, tri):
    cls = pt_class(X[pv], X[tri[:, 0]], X[tri[:, 1]], X[tri[:, 2]])
    d2 = np.empty(len(pv))
    with torch.no_grad():
        xp, xt = torch.from_numpy(X[pv]), torch.from_numpy(X[tri])
        for c in range(7):
            s = cls == c
            if s.any():
                d2[s] = d2_pt(xp[torch.from_numpy(s)], xt[torch.from_numpy(s)], c).numpy()
    return cls, d2


def ee_distance2(X, ea, eb):
    cls = ee_class(X[ea[:, 0]], X[ea[:, 1]], X[eb[:, 0]], X[eb[:, 1]])
    d2 = np.empty(len(ea))
    with torch.no_grad():
        xx = torch.from_numpy(np.stack([X[ea[:, 0]], X[ea[:, 1]], X[eb[:, 0]], X[eb[:, 1]]], axis=1))
        for c in range(9):
            s = cls == c
            if s.any():
                d2[s] = d2_ee(xx[torch.from_numpy(s)], c).numpy()
    return cls, d2


def contacts(X, F, dhat: float) -> np.ndarray:
    """Every point-triangle / edge-edge pair sharing no vertex with 0 < d < d̂: rows (term,
    class, v0, v1, v2, v3), PT = (point, triangle), EE = (edge a, edge b) with each edge's
    vertices ascending and edge a < edge b.  Candidates are exhaustive: a kd-tree ball of radius
    (primitive circumradius + d̂) around each primitive's centre holds every point / edge centre
    that can be closer than d̂."""
    from scipy.spatial import cKDTree
    F = np.asarray(F, np.int64)
    X = np.asarray(X, np.float64)
    out = []
    # point-triangle
    cen = X[F].mean(1)
    rad = np.sqrt(((X[F] - cen[:, None]) ** 2).sum(-1)).max(1)
    tree = cKDTree(X)
    lists = tree.query_ball_point(cen, rad * (1 + 1e-9) + dhat * (1 + 1e-9))
    t = np.repeat(np.arange(len(F)), [len(l) for l in lists])
    p = np.concatenate([np.asarray(l, np.int64) for l in lists]) if len(t) else np.zeros(0, np.int64)
    tri = F[t]
    keep = (tri != p[:, None]).all(1)
    p, tri = p[keep], tri[keep]
    cls, d2 = pt_distance2(X, p, tri)
    hit = (d2 < dhat * dhat) & (d2 > 0)
    out.append(np.column_stack([np.full(hit.sum(), PT), cls[hit], p[hit], tri[hit]]))
    # edge-edge
    E = _edge_ids(F)
    mid = 0.5 * (X[E[:, 0]] + X[E[:, 1]])
    half = 0.5 * np.linalg.norm(X[E[:, 1]] - X[E[:, 0]], axis=1)
    pairs = cKDTree(mid).query_pairs(2 * half.max() * (1 + 1e-9) + dhat * (1 + 1e-9), output_type="ndarray")
    pairs = np.sort(pairs, axis=1)
    a, b = E[pairs[:, 0]], E[pairs[:, 1]]
    keep = (a[:, :, None] != b[:, None, :]).all((1, 2))
    a, b = a[keep], b[keep]
    cls, d2 = ee_distance2(X, a, b)
    hit = (d2 < dhat * dhat) & (d2 > 0)
    out.append(np.column_stack([np.full(hit.sum(), EE), cls[hit], a[hit], b[hit]]))
    return np.concatenate(out).astype(np.int64)


# ------------------------------------------------------------------------------------- ACCD
def swept_pairs(X, p, F, pad: float):
    """Primitive pairs of every face pair whose swept boxes over [X, X + p], inflated by pad,
    overlap (SPEC.md:643 candidate rule): PT (point, face) and EE (edge vertices) rows."""
    F = np.asarray(F, np.int64)
    Y = X + p
    lo = np.minimum(X[F].min(1), Y[F].min(1)) - pad
    hi = np.maximum(X[F].max(1), Y[F].max(1)) + pad
    I, J = np.triu_indices(len(F), 1)
    ov = np.all((lo[I] <= hi[J]) & (lo[J] <= hi[I]), axis=1)
    I, J = I[ov], J[ov]
    pt, ee = set(), set()
    for fa, fb in zip(I.tolist(), J.tolist()):
        A, Bf = F[fa].tolist(), F[fb].tolist()
        for P_, T_, tf in ((A, Bf, fb), (Bf, A, fa)):
            for v in P_:
                if v not in T_:
                    pt.add((v, tf))
        for x in range(3):
            e1 = tuple(sorted((A[x], A[(x + 1) % 3])))
            for y in range(3):
                e2 = tuple(sorted((Bf[y], Bf[(y + 1) % 3])))
                if set(e1) & set(e2):
                    continue
                ee.add(tuple(sorted((e1, e2))))
    ptv = np.array([(v, *F[f]) for v, f in sorted(pt)], np.int64).reshape(-1, 4)
    eev = np.array([(*a, *b) for a, b in sorted(ee)], np.int64).reshape(-1, 4)
    return ptv, eev


def accd(X, p, quads: np.ndarray, edge_edge: bool, margin: float) -> np.ndarray:
    """Conservative advancement per primitive pair: t advances by
    0.9 (d - margin') / (max centred displacement of each primitive, summed) until d <= margin'
    or t >= 1; margin' = min(margin, 0.1 d(X)); at most 64 advancements."""
    if len(quads) == 0:
        return np.ones(0)
    x, d = X[quads], p[quads]  # (n, 4, 3)
    cen = d - d.mean(1, keepdims=True)
    ln = np.sqrt((cen * cen).sum(-1))
    grp = (np.array([1, 1, 0, 0], bool) if edge_edge else np.array([1, 0, 0, 0], bool))
    lp = ln[:, grp].max(1) + ln[:, ~grp].max(1)

    def dist(y):
        if edge_edge:
            _, d2 = ee_distance2(y.reshape(-1, 3), np.arange(0, 4 * len(y), 4)[:, None] + [0, 1],
                                 np.arange(0, 4 * len(y), 4)[:, None] + [2, 3])
        else:
            _, d2 = pt_distance2(y.reshape(-1, 3), np.arange(0, 4 * len(y), 4),
                                 np.arange(0, 4 * len(y), 4)[:, None] + [1, 2, 3])
        return np.sqrt(np.maximum(d2, 0.0))

    mg = np.minimum(margin, 0.1 * dist(x))
    t = np.zeros(len(x))
    done = ~(lp > 0)
    res = np.where(done, 1.0, 0.0)
    for _ in range(64):
        act = ~done
        if not act.any():
            break
        y = x[act] + t[act, None, None] * d[act]
        dd = dist(y)
        idx = np.nonzero(act)[0]
        stop = dd <= mg[act]
        res[idx[stop]] = t[idx[stop]]
        done[idx[stop]] = True
        go = idx[~stop]
        t[go] = t[go] + 0.9 * (dd[~stop] - mg[go]) / lp[go]
        over = go[t[go] >= 1.0]
        res[over] = 1.0
        done[over] = True
    res[~done] = t[~done]
    return res
