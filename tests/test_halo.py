"""Host-side checks of the tolerance-halo comparison (tests/halo.py) on the CPU oracle:
two localizations of slightly different fields agree outside the halo, and a set that
differs far from any ambiguous node is caught."""
import numpy as np
import pytest

from oracle import oracle as O

from . import halo as H


@pytest.fixture(scope="module")
def runs():
    caps = O.gen_capsules(42)
    a = O.extract_progressive(O.Analytic(caps, 0.02, threads=4), 8, 3, level_sets=True)
    # a field perturbed by ~1e-6: decisions may only flip where a value is within tol of 0.5
    b = O.extract_progressive(O.Analytic(caps, 0.02 * (1 + 3e-5), threads=4), 8, 3, level_sets=True)
    return a, b


def test_level_sets_match_counts(runs):
    a, _ = runs
    for l in range(4):
        assert len(a["evaluated_sets"][l]) == a["evals_per_level"][l]
        assert len(a["refined_sets"][l]) == a["refined_cells_per_level"][l]
        assert np.all(np.diff(a["evaluated_sets"][l].astype(np.int64)) > 0)


def test_perturbed_field_agrees_outside_halo(runs):
    a, b = runs
    halo = H.build_halo(a["evaluated_sets"], b["evaluated_sets"], a["values"], b["values"], 3, 8, 1e-4)
    H.compare_outside_halo(a["evaluated_sets"], b["evaluated_sets"], a["refined_sets"], b["refined_sets"], halo, 3, 8)
    ra = O.render_first_crossing(a["values"], 64, O.camera_from_angles(90, 0), 128, 128)
    rb = O.render_first_crossing(b["values"], 64, O.camera_from_angles(90, 0), 128, 128)
    out = ~H.ray_touches_halo_yaw90(halo, 128, 128)
    assert np.array_equal(ra["surface_k"][out], rb["surface_k"][out])


def test_difference_far_from_halo_is_caught(runs):
    a, _ = runs
    b_sets = [s.copy() for s in a["evaluated_sets"]]
    b_sets[3] = b_sets[3][1:]  # drop one level-3 evaluation: identical values => empty halo
    halo = H.build_halo(a["evaluated_sets"], b_sets, a["values"], a["values"], 3, 8, 0.0)
    with pytest.raises(AssertionError):
        H.compare_outside_halo(a["evaluated_sets"], b_sets, a["refined_sets"], a["refined_sets"], np.zeros_like(halo),
                               3, 8)
    b_ref = [s.copy() for s in a["refined_sets"]]
    b_ref[2] = b_ref[2][1:]
    with pytest.raises(AssertionError):
        H.compare_outside_halo(a["evaluated_sets"], a["evaluated_sets"], a["refined_sets"], b_ref,
                               np.zeros_like(halo), 3, 8)
