"""rtucker_verify_suite (ref capi.cpp:364-403, verify.cpp:85-416): the reference's four
property suites, with its check names and bounds, run against the GPU routines."""
import ctypes as C
import json

import pytest

pytestmark = pytest.mark.gpu

CHECKS = {
    "leverage": {"svd_form_vs_pinv_form", "effective_dimension_vs_singular_sum",
                 "effective_dimension_at_most_rank", "augmented_design_equality",
                 "scores_nonnegative", "ridge_at_most_classical", "classical_at_most_one",
                 "sum_squared_cross_equality_at_zero", "sum_squared_cross_below_score"},
    "kronecker": {"factored_scores_vs_materialized", "ridge_cross_scores_vs_materialized",
                  "cross_matrix_eigenvalue_formula"},
    "missing": {"woodbury_update_vs_recomputation", "bound_dominates_exact",
                "scores_never_decrease", "sum_squared_cross_equality_at_zero",
                "sum_squared_cross_below_score", "kronecker_coefficient_dominates"},
    "structural": {"subspace_embedding_hit_rate", "matrix_multiplication_variance_bound"},
}


def run_suite(rt, name, seed):
    passed = C.c_int(-1)
    rep = C.c_char_p()
    rc = rt.lib.rtucker_verify_suite(name.encode(), seed, C.byref(passed), C.byref(rep))
    assert rc == rt.OK, rt.lib.rtucker_last_error().decode()
    report = json.loads(rep.value.decode())
    rt.lib.rtucker_string_free(rep)
    return passed.value, report


@pytest.mark.parametrize("seed", [7, 2024])
def test_all_suites_pass(rt, seed):
    passed, report = run_suite(rt, "all", seed)
    assert [s["suite"] for s in report] == list(CHECKS)
    for s in report:
        names = {c["name"] for c in s["checks"]}
        assert names == CHECKS[s["suite"]], (s["suite"], names)
        for c in s["checks"]:
            assert c["passed"], (s["suite"], c)
        assert s["passed"] and s["elapsed_seconds"] > 0
    assert passed == 1


def test_unknown_suite_is_invalid_argument(rt):
    passed = C.c_int(-1)
    rc = rt.lib.rtucker_verify_suite(b"nope", 7, C.byref(passed), None)
    assert rc == rt.ERR_INVALID_ARGUMENT
