import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


SPEC_FIELDS = ("n", "c_i", "h_i", "w_i", "c_o", "h_f", "w_f", "stride_h", "stride_w",
               "pad_h", "pad_w", "dilation_h", "dilation_w")


def spec_from_vec(v):
    from paper_2110_03901_b200 import ConvSpec
    return ConvSpec(**{f: int(x) for f, x in zip(SPEC_FIELDS, v)})


def conv_args(spec):
    return (spec.stride_h, spec.stride_w, spec.pad_h, spec.pad_w, spec.dilation_h, spec.dilation_w)


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
