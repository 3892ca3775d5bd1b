"""Ingest parity: every format of the reference's load_mesh (binary and
ASCII STL with the weld, binary / ASCII / variable-list PLY, OBJ with polygons, relative indices
and /vt/vn suffixes) against the reference's own loader (golden vectors from oracle/_ref,
tests/golden/make_golden_ingest.py), the oracle's STL restatement on CPU, and the library's
loaders (pamopt_cu_load_stl / _load_ply / _load_obj / pamopt_cu_normalize_unit_cube)."""
import os
import struct
import tempfile

import numpy as np
import pytest

from tests.ingest_corpus import corpus, ply_bytes, stl_bytes

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_ingest.npz"))


def _stats(st):
    return [st["degenerate_faces_dropped"], st["polygons_triangulated"], st["vertices_welded"]]


def test_oracle_stl_weld_matches_reference(oracle):
    for name, (ext, data) in corpus().items():
        if ext != "stl" or data.startswith(b"solid"):  # the oracle restates the binary weld only
            continue
        v, f, st = oracle.load_stl_binary(data)
        assert np.array_equal(v.view(np.uint64), GOLD[f"{name}_v_bits"]), name
        assert np.array_equal(f, GOLD[f"{name}_f"]) and _stats(st) == list(GOLD[f"{name}_stats"]), name


def test_live_reference_matches_golden(oracle):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (no /root/reference)")
    for name, (ext, data) in corpus().items():
        with tempfile.NamedTemporaryFile(suffix="." + ext, delete=False) as fh:
            fh.write(data)
            path = fh.name
        try:
            v, f, st = oracle.ref_load_mesh(path)
        finally:
            os.unlink(path)
        assert np.array_equal(v.view(np.uint64), GOLD[f"{name}_v_bits"]) and np.array_equal(f, GOLD[f"{name}_f"]), name


@pytest.mark.gpu
def test_gpu_loaders_match_reference(api):
    for name, (ext, data) in corpus().items():
        m, st = api.load_mesh_bytes(data, ext)
        v, f = m.download()
        assert np.array_equal(v.view(np.uint64), GOLD[f"{name}_v_bits"]), name
        assert np.array_equal(f, GOLD[f"{name}_f"]), name
        assert _stats(st) == list(GOLD[f"{name}_stats"]), name


@pytest.mark.gpu
def test_gpu_loader_errors(api):
    """Malformed / truncated / empty files raise (PAMOPT_CU_EIO = the reference's
    std::runtime_error, mesh_io.cpp:17-21), for every format."""
    from paper_2509_05595_b200._lib import EIO, PamoptError
    from paper_2509_05595_b200 import fixtures as FX
    v, f = FX.icosphere(1)
    bad = [("stl", b"solid x\n facet normal 0 0 1\n"),                    # ascii stl without vertices
           ("stl", b"solid x\n facet normal 0 0 1\n outer loop\n vertex 0 0 0\n vertex 1 0 0\n"),  # dangling
           ("stl", b"solid x\n facet\n vertex 0 0 zero\n"),               # malformed vertex
           ("stl", stl_bytes(v, f)[:-30]),                                 # truncated
           ("stl", stl_bytes(v, f[:0])),                                   # no faces
           ("ply", ply_bytes(v, f).replace(b"binary_little_endian", b"ascii               ")),
           ("ply", ply_bytes(v, np.where(f == 0, 999, f))),                # index out of range
           ("ply", b"plx\nformat ascii 1.0\nend_header\n"),               # missing magic
           ("obj", b"v 1 2\nf 1 1 1\n"),                                   # malformed vertex
           ("obj", b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 4\n"),              # index out of range
           ("obj", b"v 0 0 0\nv 1 0 0\nf 1 2\n"),                          # fewer than 3 vertices
           ("obj", b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 x\n"),              # malformed index
           ("obj", b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 1 2\n")]              # only degenerate -> empty
    for ext, data in bad:
        with pytest.raises(PamoptError) as e:
            api.load_mesh_bytes(data, ext)
        assert e.value.code == EIO, (ext, data[:40])
    # a binary PLY whose face list is a quad is valid (variable lists are decoded record by record)
    quad = bytearray(ply_bytes(v, f, extras=False))
    body = quad.index(b"end_header\n") + len(b"end_header\n") + 24 * len(v)
    quad[body] = 4
    with pytest.raises(PamoptError):  # ... but 4 indices read from a 3-index record run off the end
        api.load_mesh_bytes(bytes(quad), "ply")


@pytest.mark.gpu
def test_gpu_normalize_matches_reference(api):
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_normalize.npz"))
    f = np.zeros((1, 3), np.int32)
    m = api.DeviceMesh.upload(g["v_in"], f)
    scale, tr = api.normalize_unit_cube(m, 6.0 / 128)
    v, _ = m.download()
    assert np.array_equal(v.view(np.uint64), g["v_out"].view(np.uint64))
    assert np.array_equal(np.array([scale, *tr]).view(np.uint64), g["st"].view(np.uint64))


@pytest.mark.gpu
def test_gpu_stl_large_weld(api, oracle):
    """C3-scale soup written as STL: 3M corners welded on the GPU == the oracle restatement."""
    from paper_2509_05595_b200 import fixtures as FX
    v, f, _, _ = FX.make_config("c2")
    data = stl_bytes(v, f)
    m, st = api.load_mesh_bytes(data, "stl")
    gv, gf = m.download()
    ov, of, ost = oracle.load_stl_binary(data)
    assert np.array_equal(gv.view(np.uint64), ov.view(np.uint64)) and np.array_equal(gf, of) and st == ost
    _ = struct
