"""the reference's DES with B200-calibrated GpuSpecs (tests/des_crossval.py)
against the measured C5 sweep.  CPU-only; needs oracle/_ref (the reference compiled in place)."""
import pytest

from oracle import pyoracle as O
from tests import des_crossval as X

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_b200_tile_selection_matches_survey_probe():
    # with B200-calibrated rates C1 -> 4/SM, C2 B=8 -> 2/SM, B >= 16 -> 4/SM
    g = X.gpu_spec(*X.peaks())
    c1 = O.ref_des_predict(X.SHAPE, (512, 2048, 1536), [2048] * 8, g)
    assert c1["ctas_per_sm"] == 4
    for b, want in ((8, 2), (16, 4), (32, 4), (64, 4)):
        assert X.predict(g, 1024, 16384, b)["ctas_per_sm"] == want


@needs_ref
def test_des_is_deterministic_and_bounded_by_its_roofline():
    g = X.gpu_spec(*X.peaks())
    a, b = X.predict(g, 1024, 16384, 64), X.predict(g, 1024, 16384, 64)
    assert a == b
    assert a["fused_best"] >= a["oracle_runtime"] * (1 - 1e-9)
    assert a["serial"] >= max(a["prefill_alone"], a["decode_alone"])


@needs_ref
def test_measured_calibration_predicts_the_b200_speedups():
    r = X.crossval(X.load_points())
    # fitted at one point (C2 B=64 role-alone times), the DES predicts fused-vs-serial on the
    # other 35 sweep points within 10 % on average, and better than the peak calibration
    assert r["mape_speedup_meas"] < 0.10
    assert r["mape_speedup_meas"] < r["mape_speedup_peak"]
    assert r["rank_speedup_meas"] > 0.7
