import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpamopt_cu.so")


def _have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _have_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle import pyoracle
    if not os.path.exists(os.path.join(pyoracle.HERE, "liboracle.so")):
        pyoracle.build(ref=False)
    pyoracle.set_workers(os.cpu_count() or 1)
    return pyoracle


@pytest.fixture(scope="session")
def api():
    from paper_2509_05595_b200 import api as A
    return A


@pytest.fixture(scope="session")
def c1(oracle):
    """C1 inputs and the oracle's stage outputs (cached for the session)."""
    from paper_2509_05595_b200 import fixtures as FX
    v, f, R, target = FX.make_config("c1")
    udf, sdf = oracle.compute_udf_sdf(v, f, R)
    dmc = oracle.dmc_extract(sdf, R)
    return dict(v=v, f=f, R=R, target=target, udf=udf, sdf=sdf, dmc=dmc)
