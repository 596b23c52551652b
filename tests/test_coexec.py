"""Co-execution efficiency model against golden
values of the reference (coexec.py:258-323)."""

import json
import warnings

import pytest

from conftest import GOLDEN
from paper_2005_05899_b200 import coexec as cx

ROWS = json.loads((GOLDEN / "reference_coexec.json").read_text())["rows"]


@pytest.mark.parametrize("row", ROWS, ids=lambda r: f"s{r['speedup']}-c{r['n_core']}-g{r['n_gpu']}")
def test_matches_reference(row):
    p = cx.EfficiencyParams.from_counts(row["n_core"], row["n_gpu"], row["speedup"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        assert cx.eff_core(p) == row["eff_core"]
        assert cx.eff_gpu(p) == row["eff_gpu"]
        assert cx.eff_coex1(p) == row["eff_coex1"]
        assert cx.eff_coex2(p) == row["eff_coex2"]
        for c in (1, 2):
            if row[f"red{c}"] is None:
                with pytest.raises(ValueError):
                    cx.predicted_time_reduction(p, c)
            else:
                assert cx.predicted_time_reduction(p, c) == row[f"red{c}"]


def test_validation_and_report():
    with pytest.raises(ValueError):
        cx.EfficiencyParams(speedup=0.0, ratio=1.0)
    with pytest.raises(ValueError):
        cx.EfficiencyParams.from_counts(0, 1, 2.0)
    with pytest.raises(ValueError):
        cx.predicted_time_reduction(cx.EfficiencyParams(2.0, 0.5), 3)
    with pytest.warns(UserWarning):
        cx.eff_coex2(cx.EfficiencyParams(1.5, 0.5))
    p = cx.measured_params(2237.7, 0.0555, n_core=16, n_gpu=1)
    r = cx.report(p)
    assert r["speedup"] == pytest.approx(2237.7 / 0.0555)
    assert r["eff_gpu"] + r["eff_core"] == pytest.approx(1.0)
    assert 0 < r["time_reduction_coex1"] < 1e-3  # a B200 dwarfs 16 host cores: co-execution buys nothing
