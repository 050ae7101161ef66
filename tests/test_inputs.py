"""Seeded input generator: determinism and the realised value laws."""
import numpy as np
import pytest

from nef_inputs import CONFIGS, generate_numpy


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_deterministic_and_shapes(name):
    a = generate_numpy(name)
    b = generate_numpy(name)
    assert np.array_equal(a["Y"], b["Y"])
    assert (a["mask"] is None) == (b["mask"] is None)
    if a["mask"] is not None:
        assert np.array_equal(a["mask"], b["mask"])
        assert a["mask"].dtype == np.uint8
    for x, y in zip(a["init"], b["init"]):
        assert np.array_equal(x, y) and x.dtype == np.float32
        assert x.min() >= 0.1 and x.max() <= 1.0
    assert a["Y"].dtype == np.float32 and np.all(a["Y"] >= 0)
    assert a["Y"].shape == CONFIGS[name].small_shape


def test_realised_laws():
    c3 = generate_numpy("c3")
    assert abs((c3["Y"] == 0).mean() - 0.70) < 0.03          # reading R13: ~70% zeros
    assert abs((c3["mask"] == 0).mean() - 0.20) < 0.01
    c2 = generate_numpy("c2")
    assert abs((c2["mask"] == 0).mean() - 0.10) < 0.01
    c5 = generate_numpy("c5")
    assert abs((c5["mask"] == 0).mean() - 0.05) < 0.01
    c1 = generate_numpy("c1")
    assert np.all(c1["Y"] == np.round(c1["Y"]))                # Poisson counts
    assert c1["mask"] is None


def test_beta_convention_mapping():
    """SURVEY F1 / reading R1: paper beta = BASELINE.json beta - 1."""
    for c in CONFIGS.values():
        assert c.beta == c.beta_json - 1.0
