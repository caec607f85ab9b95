import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_1710_07565_b200", "librhg_b200.so")
    orc = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(orc):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1710_07565_b200", "csrc")], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def oracle():
    from oracle.refbind import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def golden():
    import json
    d = os.path.join(ROOT, "tests", "golden")
    return {k: json.load(open(os.path.join(d, k + ".json"))) for k in ("known_answers", "layouts", "points", "stats")}
