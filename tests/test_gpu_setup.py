"""Device-side setup (§8f #2): node classification on the device
(kfbi_classify_nodes) gives the host path's flags and crossing records bit
for bit (grid.py:122-256 of the reference)."""

import os

import numpy as np
import pytest

import paper_2404_14864_b200 as k
from conftest import BOX, PI_BOX

pytestmark = pytest.mark.gpu

CASES = [
    (BOX, 128, k.CircleCurve(1.0)),
    (BOX, 1024, k.CircleCurve(1.1, center=(0.05, -0.1))),
    (BOX, 4096, k.StarCurve(1.0, c=0.2, lobes=8)),
    (BOX, 4096, k.EllipseCurve(1.2, 0.8)),
    (PI_BOX, 4096, k.StarCurve(1.5, c=0.2, lobes=3)),
    (BOX, 2048, k.StarCurve(1.0, c=0.2, lobes=5)),
]


def _host(box, m, curve):
    os.environ["KFBI_HOST_SETUP"] = "1"
    try:
        return k.build_grid(box, m, curve)
    finally:
        del os.environ["KFBI_HOST_SETUP"]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[2].kind}{c[1]}")
def test_device_classification_matches_host(case):
    box, m, curve = case
    dev = k.build_grid(box, m, curve)
    assert dev.classification._level is None          # flags came from the device
    host = _host(box, m, curve)
    assert np.array_equal(dev.classification.interior, host.classification.interior)
    assert np.array_equal(dev.classification.irregular, host.classification.irregular)
    r1, r2 = dev.records, host.records
    for name in ("owner_flat", "arm", "x", "y", "theta", "d", "owner_interior"):
        assert np.array_equal(getattr(r1, name), getattr(r2, name)), name
    assert np.array_equal(dev.edge_theta, host.edge_theta)
    # level on demand equals the host level
    if m <= 1024:
        assert np.array_equal(dev.classification.level, host.classification.level)
