import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (str(ROOT), str(ROOT / "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)
# The unmodified reference (iota-sim), installed by __graft_entry__.build() into the
# git-ignored baseline/_ref (it travels to the GPU box with the snapshot).  On the path,
# the drop-in's errors and result types ARE the reference's (errors.py, butterfly.py).
REF = ROOT / "baseline" / "_ref"
if (REF / "iota_sim").is_dir() and str(REF) not in sys.path:
    sys.path.append(str(REF))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: larger parity sweeps")


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
