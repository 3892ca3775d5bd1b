"""Synthetic STL / PLY files for the ingest parity tests (written deterministically, so the GPU
box regenerates the same bytes)."""
import struct

import numpy as np

from paper_2509_05595_b200 import fixtures as FX


def stl_bytes(v, f, extra_degenerate=0, nan_corner=False):
    """Binary STL of faces f over vertices v (one 50-byte record per facet, float32 corners)."""
    tris = [v[t] for t in f]
    for k in range(extra_degenerate):  # facets with two identical corners -> dropped after welding
        a = v[f[k, 0]]
        tris.append(np.stack([a, a, v[f[k, 1]]]))
    if nan_corner:
        tris.append(np.array([[np.nan, 0.0, 0.0], [1.0, 2.0, 3.0], [1.0, 2.0, 4.0]]))
        tris.append(np.array([[np.nan, 0.0, 0.0], [1.0, 2.0, 3.0], [1.0, 3.0, 3.0]]))
    out = bytearray(b"binary stl written by tests/ingest_corpus.py".ljust(80, b" "))
    out += struct.pack("<I", len(tris))
    for t in tris:
        n = np.zeros(3, np.float32)
        out += n.tobytes() + np.asarray(t, np.float32).tobytes() + b"\0\0"
    return bytes(out)


def ply_bytes(v, f, double=True, extras=True):
    """Binary little-endian PLY: x/y/z (+ a float normal and a uchar colour), face lists uchar/int
    (+ a trailing int face property)."""
    vt = "double" if double else "float"
    hdr = ["ply", "format binary_little_endian 1.0", "comment ingest_corpus", f"element vertex {len(v)}",
           f"property {vt} x", f"property {vt} y", f"property {vt} z"]
    if extras:
        hdr += ["property float nx", "property uchar red"]
    hdr += [f"element face {len(f)}", "property list uchar int vertex_indices"]
    if extras:
        hdr += ["property int tag"]
    hdr += ["end_header"]
    out = bytearray(("\n".join(hdr) + "\n").encode())
    dt = np.float64 if double else np.float32
    for i, p in enumerate(v):
        out += np.asarray(p, dt).tobytes()
        if extras:
            out += struct.pack("<fB", 0.5, i % 251)
    for i, t in enumerate(f):
        out += struct.pack("<B", 3) + np.asarray(t, np.int32).tobytes()
        if extras:
            out += struct.pack("<i", i)
    return bytes(out)


def fmt(x: float) -> str:
    return repr(float(x))  # shortest round-trip text: the loaders must recover the same double


def obj_bytes(v, polys, rel_from=None, suffix=False, comments=True):
    """OBJ text: 'v x y z' lines, then 'f' lines of 1-based indices (negative / relative from
    face `rel_from` on), '/vt/vn' suffixes when `suffix`, comments and blank lines."""
    lines = ["# written by tests/ingest_corpus.py", ""] if comments else []
    lines += [f"v {fmt(p[0])} {fmt(p[1])}   {fmt(p[2])}" for p in v]
    for i, poly in enumerate(polys):
        toks = []
        for k, x in enumerate(poly):
            x = int(x)
            t = str(x - len(v)) if rel_from is not None and i >= rel_from else str(x + 1)
            if suffix and k % 2 == 0:
                t += f"/{x + 1}/{x + 1}" if k % 4 == 0 else f"//{x + 1}"
            toks.append(t)
        lines.append("f " + " ".join(toks))
    return ("\n".join(lines) + "\n").encode()


def ply_ascii_bytes(v, polys):
    hdr = ["ply", "format ascii 1.0", "comment text body", f"element vertex {len(v)}", "property double x",
           "property double y", "property double z", "property uchar red", f"element face {len(polys)}",
           "property list uchar int vertex_indices", "end_header"]
    body = [f"{fmt(p[0])} {fmt(p[1])} {fmt(p[2])} {i % 200}" for i, p in enumerate(v)]
    body += [" ".join([str(len(pl))] + [str(int(x)) for x in pl]) for pl in polys]
    return ("\n".join(hdr + body) + "\n").encode()


def ply_varlist_bytes(v, polys):
    """Binary little-endian PLY with variable-length face lists (quads, pentagons)."""
    hdr = ["ply", "format binary_little_endian 1.0", f"element vertex {len(v)}", "property float x",
           "property float y", "property float z", f"element face {len(polys)}",
           "property list uchar int vertex_indices", "end_header"]
    out = bytearray(("\n".join(hdr) + "\n").encode())
    for p in v:
        out += np.asarray(p, np.float32).tobytes()
    for pl in polys:
        out += struct.pack("<B", len(pl)) + np.asarray(pl, np.int32).tobytes()
    return bytes(out)


def stl_ascii_bytes(v, f, extra_degenerate=0):
    tris = [v[t] for t in f]
    for k in range(extra_degenerate):
        a = v[f[k, 0]]
        tris.append(np.stack([a, a, v[f[k, 1]]]))
    lines = ["solid written_by_tests"]
    for t in tris:
        lines += ["  facet normal 0 0 0", "    outer loop"]
        lines += [f"      vertex {fmt(p[0])} {fmt(p[1])} {fmt(p[2])}" for p in t]
        lines += ["    endloop", "  endfacet"]
    lines.append("endsolid written_by_tests")
    return ("\n".join(lines) + "\n").encode()


def quads_of(v, f):
    """Merge face pairs sharing an edge into quads (and a few pentagons) for polygon tests."""
    polys, used = [], np.zeros(len(f), bool)
    edge = {}
    for i, t in enumerate(f.tolist()):
        for k in range(3):
            edge.setdefault((t[(k + 1) % 3], t[k]), i)
    for i, t in enumerate(f.tolist()):
        if used[i]:
            continue
        j = edge.get((t[0], t[1]))
        if j is not None and not used[j] and j != i and i % 3 == 0:
            u = f[j].tolist()
            opp = [x for x in u if x not in (t[0], t[1])][0]
            polys.append([t[0], opp, t[1], t[2]])
            used[i] = used[j] = True
        else:
            polys.append(t)
            used[i] = True
    return polys


def corpus():
    """name -> (extension, bytes)."""
    out = {}
    v, f = FX.icosphere(3)
    out["ico_stl"] = ("stl", stl_bytes(v, f, extra_degenerate=5))
    out["nan_stl"] = ("stl", stl_bytes(v[:40] * 3.0, f[:20] % 40, nan_corner=True))
    vs, fs = FX.soup(2, 5000, seed=4)
    out["soup_stl"] = ("stl", stl_bytes(vs, fs))
    df = f.copy()
    df[:4, 2] = df[:4, 1]  # degenerate faces in the index list
    out["ico_ply_double"] = ("ply", ply_bytes(v, df, double=True, extras=True))
    out["ico_ply_float"] = ("ply", ply_bytes(v, f, double=False, extras=False))
    # text formats and variable-length polygon lists
    rng = np.random.default_rng(9)
    vn = v * (1.0 + 0.01 * rng.standard_normal(len(v)))[:, None]
    polys = quads_of(vn, f)
    polys.append([0, 0, 1])                      # degenerate triangle (dropped)
    polys.append([1, 2, 3, 4, 5])                # pentagon (fanned)
    out["ico_obj"] = ("obj", obj_bytes(vn, polys, rel_from=len(polys) // 2, suffix=True))
    out["ico_ply_ascii"] = ("ply", ply_ascii_bytes(vn, polys))
    out["ico_ply_varlist"] = ("ply", ply_varlist_bytes(vn, polys))
    out["ico_stl_ascii"] = ("stl", stl_ascii_bytes(vn, f, extra_degenerate=3))
    return out
