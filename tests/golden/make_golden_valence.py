"""Generates tests/golden/ref_link_valence.npz: the REFERENCE's own link_condition_holds
(mesh.cpp:301-358, compiled in place into oracle/_ref by `make -C oracle ref`) on meshes whose
vertex valence far exceeds any fixed per-thread buffer: a closed bipyramid with a 1000-valent
apex pair, an open 600-triangle fan (boundary apex) and a bipyramid whose equator is split by a
diagonal strip.  Every edge of each mesh is queried.

    python tests/golden/make_golden_valence.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle as O  # noqa: E402


def bipyramid(n: int, h: float = 1.0):
    t = 2 * np.pi * np.arange(n) / n
    ring = np.stack([np.cos(t), np.sin(t), 0.05 * np.sin(7 * t)], 1)
    v = np.concatenate([ring, [[0, 0, h], [0, 0, -h]]])
    top, bot = n, n + 1
    f = [[i, (i + 1) % n, top] for i in range(n)] + [[(i + 1) % n, i, bot] for i in range(n)]
    return v, np.array(f, np.int32)


def fan(n: int):
    t = 2 * np.pi * np.arange(n + 1) / (n + 1) * 0.9
    ring = np.stack([np.cos(t), np.sin(t), 0.1 * np.cos(3 * t)], 1)
    v = np.concatenate([ring, [[0, 0, 0.3]]])
    f = [[i, i + 1, n + 1] for i in range(n)]
    return v, np.array(f, np.int32)


def edges_of(f):
    e = np.sort(np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]]), axis=1)
    return np.unique(e, axis=0).astype(np.int32)


def meshes():
    return {"bipyramid1000": bipyramid(1000), "fan600": fan(600), "bipyramid40": bipyramid(40)}


if __name__ == "__main__":
    out = {}
    for name, (v, f) in meshes().items():
        e = edges_of(f)
        out[f"{name}_v"], out[f"{name}_f"], out[f"{name}_e"] = v, f, e
        out[f"{name}_r"] = O.ref_link_condition(v, f, e).astype(np.int8)
        print(name, len(f), "faces", int(out[f"{name}_r"].sum()), "of", len(e), "edges pass")
    np.savez_compressed(os.path.join(HERE, "ref_link_valence.npz"), **out)
