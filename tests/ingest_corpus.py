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
    return out
