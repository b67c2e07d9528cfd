import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def gpu_lib():
    """The product library on a GPU box (fails loudly if missing)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2110_07029_b200 import _lib
    return _lib.load()


def pytest_sessionfinish(session, exitstatus):
    """Write the achieved parity errors (tests/_parity_log.py) next to the GPU run."""
    import json
    here = os.path.dirname(os.path.abspath(__file__))
    if here not in sys.path:
        sys.path.insert(0, here)
    import _parity_log as plog
    if not plog.RECORDS:
        return
    path = os.environ.get("PARITY_LOG", os.path.join(ROOT, "gpurun_out", "parity_errors.json"))
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump({"exitstatus": int(exitstatus), "records": plog.RECORDS}, f, indent=1)
