"""Independent exact-arithmetic triangle-triangle oracle (Python Fractions) — test-only.

Definition checked (pinned in DESIGN.md §2.3): two faces self-intersect iff
they are duplicates or either is degenerate, or their closed intersection is NOT contained in
the convex hull of the vertices they share by index (empty set for 0 shared, the point A for one
shared vertex, the segment AB for a shared edge).  The intersection is computed by exact
Sutherland-Hodgman clipping — a different algorithm from the orientation-predicate verdicts of
the oracle and the CUDA narrow phase, which must agree with it on every pair.
"""
from fractions import Fraction


def _sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def _lerp(p, q, t):
    return (p[0] + t * (q[0] - p[0]), p[1] + t * (q[1] - p[1]), p[2] + t * (q[2] - p[2]))


def _clip(poly, P, m, sgn_ref):
    """Keep the closed side of the plane {X : m.(X-P) has sign sgn_ref or 0}."""
    if not poly:
        return poly
    out = []
    n = len(poly)
    for i in range(n):
        cur, nxt = poly[i], poly[(i + 1) % n]
        dc = _dot(m, _sub(cur, P)) * sgn_ref
        dn = _dot(m, _sub(nxt, P)) * sgn_ref
        if dc >= 0:
            out.append(cur)
        if (dc > 0 and dn < 0) or (dc < 0 and dn > 0):
            out.append(_lerp(cur, nxt, dc / (dc - dn)))
    # dedupe consecutive duplicates
    ded = []
    for p in out:
        if not ded or ded[-1] != p:
            ded.append(p)
    if len(ded) > 1 and ded[0] == ded[-1]:
        ded.pop()
    return ded


def _sign(x):
    return (x > 0) - (x < 0)


def intersect(T1, T2, shared_idx1, shared_idx2):
    """T1, T2: 3 points (float triples).  shared_idx1[k] = index into T2 of T1's vertex k or -1."""
    T1 = [tuple(Fraction(c) for c in p) for p in T1]
    T2 = [tuple(Fraction(c) for c in p) for p in T2]
    ns = sum(1 for s in shared_idx1 if s >= 0)
    if ns == 3:
        return True
    n1 = _cross(_sub(T1[1], T1[0]), _sub(T1[2], T1[0]))
    n2 = _cross(_sub(T2[1], T2[0]), _sub(T2[2], T2[0]))
    if n1 == (0, 0, 0) or n2 == (0, 0, 0):
        return True
    d = [_dot(n2, _sub(p, T2[0])) for p in T1]
    if all(x == 0 for x in d):
        poly = list(T1)  # coplanar
    else:
        pts = []
        for i in range(3):
            j = (i + 1) % 3
            if d[i] == 0:
                pts.append(T1[i])
            if d[i] * d[j] < 0:
                pts.append(_lerp(T1[i], T1[j], d[i] / (d[i] - d[j])))
        poly = []
        for p in pts:
            if p not in poly:
                poly.append(p)
    for k in range(3):
        P, Q, Rr = T2[k], T2[(k + 1) % 3], T2[(k + 2) % 3]
        m = _cross(_sub(Q, P), n2)
        s = _sign(_dot(m, _sub(Rr, P)))
        poly = _clip(poly, P, m, s)
        if not poly:
            return False
    shared = [T1[k] for k in range(3) if shared_idx1[k] >= 0]
    if ns == 0:
        return True
    if ns == 1:
        A = shared[0]
        return any(p != A for p in poly)
    A, B = shared
    AB = _sub(B, A)
    for p in poly:
        ap = _sub(p, A)
        if _cross(AB, ap) != (0, 0, 0):
            return True
        t = _dot(ap, AB)
        if t < 0 or t > _dot(AB, AB):
            return True
    return False


def verdict_pairs(v, f, pairs):
    out = []
    for a, b in pairs:
        t1, t2 = f[a], f[b]
        s1 = [next((j for j in range(3) if t1[k] == t2[j]), -1) for k in range(3)]
        s2 = [next((k for k in range(3) if t1[k] == t2[j]), -1) for j in range(3)]
        out.append(1 if intersect([v[i] for i in t1], [v[i] for i in t2], s1, s2) else 0)
    return out


def classify_pairs(v, f, pairs):
    """classify_pair in exact rationals: (shared count by index, coplanar), a
    degenerate face counting as coplanar."""
    sh, cp = [], []
    for a, b in pairs:
        t1, t2 = f[a], f[b]
        ns = sum(1 for k in range(3) if t1[k] in t2)
        T1 = [tuple(Fraction(c) for c in v[i]) for i in t1]
        T2 = [tuple(Fraction(c) for c in v[i]) for i in t2]
        n1 = _cross(_sub(T1[1], T1[0]), _sub(T1[2], T1[0]))
        n2 = _cross(_sub(T2[1], T2[0]), _sub(T2[2], T2[0]))
        if ns == 3 or n1 == (0, 0, 0) or n2 == (0, 0, 0):
            c = 1
        else:
            c = int(all(_dot(n1, _sub(p, T1[0])) == 0 for p in T2))
        sh.append(ns)
        cp.append(c)
    return sh, cp
