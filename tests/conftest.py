import os
import sys
from pathlib import Path

import pytest

# The single-device loopback of the multi-GPU ring runs every rank's streams on one GPU;
# the chunked executor's streams wait on flags (cuStreamWaitValue32), which must not
# share a hardware queue with the work that writes them: one queue per stream (set before
# the CUDA context exists).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

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
