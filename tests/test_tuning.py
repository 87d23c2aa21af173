"""GPU tuner: grid validation, selection rule, feasibility, determinism (the
reference's tests/test_tuning.py cases, on the GPU generator)."""
import pytest

from paper_2406_15486_b200 import InfeasibleGridError, InputError
from paper_2406_15486_b200.tuning import CellResult, RangeResult, TuneGrid, TuneResult, require_feasible, tune


def test_empty_lists_rejected():
    with pytest.raises(InputError):
        TuneGrid((), (0.9,), (1,), ((64, 64),), 0.9)


def test_bad_recall():
    with pytest.raises(InputError):
        TuneGrid((0.9,), (0.9,), (1,), ((64, 64),), 1.2)


def test_bad_range():
    with pytest.raises(InputError):
        TuneGrid((0.9,), (0.9,), (1,), ((128, 64),), 0.9)


def test_require_feasible_and_json():
    cell = CellResult(1, 8, 0.9, 0.9, 1, 0.5, 0.3, False, "cra_full")
    res = TuneResult(0.9, 1, 0, (RangeResult(1, 8, False, None, (cell,)),))
    assert not res.all_feasible
    with pytest.raises(InfeasibleGridError):
        require_feasible(res)
    d = res.to_json_dict()
    assert d["ranges"][0]["best"] is None and d["ranges"][0]["grid"][0]["mean_density"] == 0.3


def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.gpu
def test_full_thresholds_always_feasible():
    _gpu()
    grid = TuneGrid((1.0,), (1.0,), (1,), ((2048, 2048),), 0.999, trials_per_cell=2)
    res = tune(grid, heads=2)
    assert res.all_feasible
    b = res.ranges[0].best
    assert (b.alpha_c, b.alpha_s, b.chunk_n) == (1.0, 1.0, 1) and b.mean_cra >= 0.999


@pytest.mark.gpu
def test_best_minimizes_density_and_recall_monotone():
    _gpu()
    grid = TuneGrid((0.7, 0.85, 0.95), (0.7, 0.95), (1, 2), ((2048, 2048),), 0.0, trials_per_cell=2)
    cells = tune(grid, heads=2).ranges[0].cells
    last = -1.0
    for target in (0.2, 0.5, 0.8, 0.9, 0.95):
        feasible = [c for c in cells if c.mean_cra >= target]
        if not feasible:
            break
        density = min(c.mean_density for c in feasible)
        assert density >= last - 1e-12
        last = density
    g2 = TuneGrid((0.7, 0.95), (0.7, 0.95), (1, 2), ((2048, 2048),), 0.3, trials_per_cell=2)
    r = tune(g2, heads=2).ranges[0]
    feasible = [c for c in r.cells if c.feasible]
    assert r.best.mean_density == min(c.mean_density for c in feasible)


@pytest.mark.gpu
def test_infeasible_range_reported_and_deterministic():
    _gpu()
    grid = TuneGrid((0.3,), (0.3,), (1,), ((4096, 4096),), 0.999, trials_per_cell=1)
    res = tune(grid, heads=2)
    assert not res.all_feasible and res.ranges[0].best is None
    with pytest.raises(InfeasibleGridError):
        require_feasible(res)
    g = TuneGrid((0.9,), (0.9,), (1, 2), ((2048, 2048),), 0.5, trials_per_cell=2)
    assert tune(g, heads=2).to_json() == tune(g, heads=2).to_json()


@pytest.mark.gpu
def test_sampled_metric_above_oracle_cap():
    _gpu()
    grid = TuneGrid((0.95,), (0.95,), (1,), ((16384, 16384),), 0.0, trials_per_cell=1)
    c = tune(grid, heads=2).ranges[0].cells[0]
    assert c.cra_metric == "cra_sampled" and 0 < c.mean_density <= 1 and 0.9 <= c.mean_cra <= 1 + 1e-9
