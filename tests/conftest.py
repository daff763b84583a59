import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as f:
        return {k: f[k] for k in f.files}


def cameras_from(g: dict, camera_cls):
    """Rebuild the fixture's cameras with the given Camera class."""
    return [
        camera_cls(fx=float(g["cam_fx"][i]), fy=float(g["cam_fy"][i]), cx=float(g["cam_cx"][i]),
                   cy=float(g["cam_cy"][i]), rotation=g["cam_R"][i], translation=g["cam_t"][i],
                   width=int(g["cam_w"][i]), height=int(g["cam_h"][i]))
        for i in range(len(g["cam_fx"]))
    ]


def rel_err(a, b) -> float:
    """max |a - b| / max(|b|, 1): the parity metric of SURVEY.md §8c."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0)))


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
