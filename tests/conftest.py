import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


def _make(target):
    r = subprocess.run(["make", "-s", "-C", ROOT, target], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"make {target} failed:\n{r.stdout}\n{r.stderr}")


def pytest_sessionstart(session):
    # CPU-side libraries (generator, oracle) are cheap to build; the CUDA library is
    # built by __graft_entry__.build() / `make`, and tests that need it build on demand.
    if not (os.path.exists(os.path.join(ROOT, "gen", "libgen.so"))
            and os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so"))):
        _make("cpu")


@pytest.fixture(scope="session")
def remoe_lib_built():
    # built here by `make` / __graft_entry__.build(); the .so travels to the GPU box
    if not os.path.exists(os.path.join(ROOT, "paper_2512_18674_b200", "libremoe.so")):
        _make("all")
    return True
