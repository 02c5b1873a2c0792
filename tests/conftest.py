import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

SPACES = os.path.join(ROOT, "spaces")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: longer CPU test")


def space_path(name):
    return os.path.join(SPACES, f"{name}.json")


def space_text(name):
    with open(space_path(name)) as fh:
        return fh.read()


def golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def oracle_spaces():
    from oracle import space as S
    return {n: S.load_space(space_path(n)) for n in ("P0", "C1", "C2", "C3", "C4", "C5")}


def cfg_digits(sp, cfg):
    """Digits of a configuration given as {name: value}; others at their default digit."""
    dg = [f.default_digit for f in sp.features]
    for k, v in cfg.items():
        j = sp.index[k]
        vals = sp.features[j].values
        dg[j] = next(i for i, x in enumerate(vals) if x == v and type(x) is type(v)) if not isinstance(v, float) \
            else next(i for i, x in enumerate(vals) if abs(float(x) - v) < 1e-12)
    return dg
