"""The CUDA path against the REFERENCE'S OWN CODE.

``oracle.ref`` binds ``oracle/_ref/libgsgp_ref.so`` — /root/reference/proj's sources compiled
unmodified against stand-in Eigen/FFTW headers (oracle/refshim/README.md) — behind the same
front-end as the restatement.  These tests re-run the core GPU parity tests of the other
files with that library as the checker (their module-level ``O`` swapped for the reference
front-end), so every bound they assert holds against the reference itself, not only against
the restatement.  The library is built in the container that has /root/reference and travels
to the GPU box prebuilt; nothing here reads /root/reference at run time.
"""
import numpy as np
import pytest

import oracle.ref as R
import paper_2101_11751_b200 as G
import test_gpu_cov as TC
import test_gpu_loglik as TL
import test_gpu_parity as TP
import test_gpu_probes as TPR

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="oracle/_ref/libgsgp_ref.so not built")]


@pytest.fixture(autouse=True)
def reference_checker(monkeypatch):
    """Every ``O.`` call of the re-used test modules goes to the reference build."""
    front = R._mod
    assert "interp.cpp" in R.ref_build_info()
    for mod in (TP, TL, TC, TPR):
        monkeypatch.setattr(mod, "O", front)
    yield


@pytest.mark.parametrize("d,scheme,dtype,sizes,n", TP.CASES)
def test_precompute_matches_reference(d, scheme, dtype, sizes, n):
    TP.test_precompute_matches_oracle(d, scheme, dtype, sizes, n)


@pytest.mark.parametrize("d,scheme", [(1, G.InterpScheme.Cubic), (2, G.InterpScheme.Cubic),
                                      (3, G.InterpScheme.Cubic), (2, G.InterpScheme.Linear)])
def test_structure_with_on_node_rows(d, scheme):
    TP.test_structure_with_on_node_rows(d, scheme)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_interp_weights_bit_exact(d):
    TP.test_interp_weights_bit_exact(d)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_classify_near_node_rows(dtype):
    TP.test_classify_near_node_rows(dtype)


def test_out_of_grid_errors_report_first_row():
    TP.test_out_of_grid_errors_report_first_row()


def test_batches_merge_and_devices():
    TP.test_batches_merge_and_devices()


@pytest.mark.parametrize("d", [1, 2, 3])
def test_operators_match_reference(d):
    TP.test_operators_match_oracle(d)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_efcg_and_posterior_mean_match_reference(d):
    TP.test_efcg_and_posterior_mean_match_oracle(d)


def test_predict_mean_bit_exact_given_coeffs():
    TP.test_predict_mean_bit_exact_given_coeffs()


def test_breakdown_and_nonconvergence():
    TP.test_breakdown_and_nonconvergence()


@pytest.mark.parametrize("cfg_id,n", [(3, 100_000), (5, 60_000), (2, 400_000), (4, 300_000)])
def test_baseline_config_prefix_matches_reference(cfg_id, n):
    TP.test_baseline_config_prefix_matches_oracle(cfg_id, n)


@pytest.mark.parametrize("d,sizes,n", [(1, (40,), 5000), (2, (16, 14), 5000), (3, (10, 9, 8), 5000)])
def test_probe_images_match_reference(d, sizes, n):
    TL.test_probe_images_match_oracle(d, sizes, n)


def test_efla_matches_reference():
    TL.test_efla_matches_oracle()


def test_loglik_matches_reference():
    TL.test_loglik_matches_oracle()


@pytest.mark.parametrize("d,sizes,ls", [(1, (60,), [0.03]), (2, (16, 14), [0.2, 0.25])])
def test_symmetric_grid_route_matches_reference(d, sizes, ls):
    TL.test_symmetric_grid_route_matches_oracle(d, sizes, ls)


@pytest.mark.parametrize("d,sizes,ls", [(1, (80,), [0.1]), (2, (20, 18), [0.2, 0.25])])
def test_dense_route_matches_reference(d, sizes, ls):
    TL.test_dense_route_matches_oracle(d, sizes, ls)


def test_auto_route_selection_matches_reference():
    TL.test_auto_route_selection_matches_oracle()


@pytest.mark.parametrize("d,sizes,ls,ns", [(1, (50,), [0.05], 9), (2, (16, 14), [0.2, 0.25], 12)])
def test_cov_exact_matches_reference(d, sizes, ls, ns):
    TC.test_cov_exact_matches_oracle(d, sizes, ls, ns)


@pytest.mark.parametrize("rank", [5, 30])
def test_cov_lowrank_matches_reference(rank):
    TC.test_cov_lowrank_matches_oracle(rank)


def test_substream_probe_images_match_reference():
    TPR.test_substream_probe_images_match_oracle()
