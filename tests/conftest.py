import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libctap.so")
    config.addinivalue_line("markers", "slow: long-running GPU parity runs")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as d:
        return {k: d[k] for k in d.files}


@pytest.fixture(scope="session")
def golden():
    return load_golden


def oracle_grid(d):
    from oracle import split_step as orc

    return orc.Grid(tuple(int(v) for v in d["n"]), tuple(float(v) for v in d["extents"]),
                    tuple(float(v) for v in d["origin"]))


def product_grid(d):
    from paper_1309_2451_b200 import qgrid

    return qgrid.SimGrid(tuple(int(v) for v in d["n"]), tuple(float(v) for v in d["extents"]),
                         tuple(float(v) for v in d["origin"]))
