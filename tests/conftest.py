import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libnef.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "paper_values.json")) as f:
        return json.load(f)


@pytest.fixture
def record_err(request):
    """Record a measured parity error next to its bar: printed, and appended as a JSON line to
    $NEF_ERR_LOG when set (collected into DESIGN.md's error table)."""
    import json

    def rec(err, bar, what=""):
        line = {"test": request.node.nodeid, "what": what, "err": float(err), "bar": float(bar)}
        print("PARITY %s %s err=%.3e bar=%.1e" % (request.node.nodeid, what, err, bar))
        path = os.environ.get("NEF_ERR_LOG")
        if path:
            with open(path, "a") as f:
                f.write(json.dumps(line) + "\n")
        return err
    return rec
