"""compute_errors / dump_field against the reference's own functions
(report.py:37-62), run on the golden C1 field (CPU)."""

import os
import sys
import types

import numpy as np
import pytest

import paper_2404_14864_b200 as k
from conftest import BOX, golden


def _ref_report():
    if not os.path.isdir("/root/reference/pkg/src"):
        pytest.skip("reference not mounted (GPU box)")
    mpl = types.ModuleType("matplotlib")
    mpl.use = lambda *a, **kw: None
    plt = types.ModuleType("matplotlib.pyplot")
    mpl.pyplot = plt
    sys.modules.setdefault("matplotlib", mpl)
    sys.modules.setdefault("matplotlib.pyplot", plt)
    sys.path.insert(0, "/root/reference/pkg/src")
    import kfbi

    return kfbi


def test_compute_errors_and_dump_field_match_reference(tmp_path):
    geo = k.build_grid(BOX, 128, k.StarCurve(1.0, c=0.2, lobes=8))
    u = golden("runs")["c1_heat_flower128__u"]
    heat = k.HeatPlaneDecay(c=1.0)
    exact = lambda x, y: heat.u0(x, y) * 0.0 + heat.dirichlet(x, y, 1.0)  # noqa: E731
    mine = k.compute_errors(u, exact, geo.grid, geo.classification)
    kf = _ref_report()
    ref_geo = kf.build_grid(BOX, 128, kf.StarCurve(1.0, c=0.2, lobes=8))
    ref = kf.compute_errors(u, exact, ref_geo.grid, ref_geo.classification)
    assert mine == ref
    a = k.dump_field(u, geo.grid, geo.classification, tmp_path / "a.csv", t=1.0, equation="heat")
    b = kf.dump_field(u, ref_geo.grid, ref_geo.classification, tmp_path / "b.csv", t=1.0,
                      equation="heat")
    assert open(a).read() == open(b).read()
    uc = u * (1.0 + 0.5j)
    a = k.dump_field(uc, geo.grid, geo.classification, tmp_path / "c.csv")
    b = kf.dump_field(uc, ref_geo.grid, ref_geo.classification, tmp_path / "d.csv")
    assert open(a).read() == open(b).read()


@pytest.mark.gpu
def test_compute_errors_device_input():
    import torch

    geo = k.build_grid(BOX, 128, k.StarCurve(1.0, c=0.2, lobes=8))
    u = golden("runs")["c1_heat_flower128__u"]
    heat = k.HeatPlaneDecay(c=1.0)
    exact = lambda x, y: heat.dirichlet(x, y, 1.0)  # noqa: E731
    host = k.compute_errors(u, exact, geo.grid, geo.classification)
    dev = k.compute_errors(torch.from_numpy(u).cuda(), exact, geo.grid, geo.classification)
    assert dev[0] == host[0]
    assert abs(dev[1] - host[1]) <= 1e-14 * host[1]
