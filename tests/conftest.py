import os
import sys

# Before CUDA starts: eager module loading (the in-kernel peer-memory allreduce
# of the multi-rank tests needs every kernel loaded up front) and enough
# hardware queues that in-process ranks' streams do not serialise.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import pytest  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    d = os.path.join(ROOT, "tests", "golden")

    def load(name):
        with np.load(os.path.join(d, name + ".npz"), allow_pickle=False) as z:
            return {k: z[k] for k in z.files}

    return load


@pytest.fixture(scope="session")
def ref():
    """oracle/_ref (the reference compiled verbatim) — built here, prebuilt on the GPU box."""
    from oracle import refbind

    if not os.path.exists(refbind.LIB_PATH):
        if os.path.isdir(refbind.REF_SRC):
            refbind.build()
        else:
            pytest.skip("oracle/_ref not built and reference sources absent")
    return refbind
