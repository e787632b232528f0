import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through libihs_b200.so")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def O():
    from oracle import oracle

    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def R():
    """The reference's own headers compiled against oracle/eigen_stub (oracle/_ref/libihs_ref.so). Built here
    from /root/reference (make -C oracle ref); elsewhere the prebuilt library that travels with the repo."""
    import pathlib
    import subprocess

    from oracle import ref

    if pathlib.Path("/root/reference/proj/include/ihs").is_dir():
        subprocess.run(["make", "-s", "-C", str(pathlib.Path(ROOT) / "oracle"), "ref"], check=True)
    elif not ref.REF_LIB_PATH.exists():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return ref


@pytest.fixture(scope="session")
def ihs():
    from paper_2006_05874_b200 import ihs as m

    return m


@pytest.fixture(scope="session")
def gpu(ihs):
    # GPU tests fail loudly (no skip) when the device path is unavailable.
    n = ihs.device_count()
    assert n >= 1, "no CUDA device visible to libihs_b200.so"
    return ihs
