import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a real B200 (run with -m gpu under gpurun)")


@pytest.fixture(scope="session")
def oracle():
    from tests.cpu_checkers import load_oracle
    return load_oracle()


@pytest.fixture(scope="session")
def ref():
    from tests.cpu_checkers import load_ref, ref_available
    if not ref_available() and not os.path.isdir("/root/reference"):
        pytest.skip("oracle/_ref not built and reference sources absent")
    return load_ref()


@pytest.fixture(scope="session")
def kat():
    import json
    return json.load(open(os.path.join(ROOT, "tests", "golden", "ref_kat.json")))


@pytest.fixture(scope="session")
def seeded():
    import json
    return json.load(open(os.path.join(ROOT, "tests", "golden", "ref_seeded.json")))
