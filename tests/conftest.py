import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: large-config parity (minutes)")
    # the CPU checker and the libraries are built by __graft_entry__.build(); build here only if absent
    need = [os.path.join(ROOT, "oracle", "liboracle.so"), os.path.join(ROOT, "oracle", "liboracle_text.so"),
            os.path.join(ROOT, "paper_2407_03618_b200", "libsparselex_b200.so"),
            os.path.join(ROOT, "paper_2407_03618_b200", "libsl_synth.so")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2407_03618_b200", "csrc"), "-j4"], check=True,
                       capture_output=True)


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    return True
