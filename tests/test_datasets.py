"""Host input builders (paper_1003_3272_b200.datasets) against the reference's
own builders: bit for bit where the reference is importable in this
container, and against the input digests the golden fixtures recorded
(tests/golden/make_golden.py) everywhere.  CPU only."""

import numpy as np
import pytest

import golden_io as G
import refload
from paper_1003_3272_b200 import datasets as D


def test_c2_system_matrix_and_counts_match_the_golden_digests():
    e, y, _ = G.c2_inputs()
    gold = G.load("pet_c2")
    assert G.digest(e) == str(gold["e_digest"])
    np.testing.assert_array_equal(y, gold["y"])


def test_c3_dissimilarities_match_the_golden_digest():
    diss, _ = G.c3_inputs(3)
    assert G.digest(diss) == str(G.load("mds_c3")["diss_digest"])


ref = pytest.mark.skipif(not refload.available(), reason="reference not present")


@ref
@pytest.mark.parametrize("side,det", [(5, 8), (12, 16), (20, 24)])
def test_system_matrix_bitwise(side, det):
    R = refload.load()
    want = R.build_system_matrix(R.PetGeometry(grid_side=side, n_detectors=det))
    got = D.build_system_matrix(D.PetGeometry(side, det))
    np.testing.assert_array_equal(got, want)


@ref
@pytest.mark.parametrize("side", [1, 2, 7, 16])
def test_neighborhoods_and_phantom_bitwise(side):
    R = refload.load()
    assert [list(x) for x in D.build_neighborhoods(side)] == \
        [list(x) for x in R.build_neighborhoods(side)]
    np.testing.assert_array_equal(D.default_phantom(side), R.default_phantom(side))


@ref
def test_simulate_counts_bitwise():
    R = refload.load()
    geo = R.PetGeometry(grid_side=10, n_detectors=12)
    e = R.build_system_matrix(geo)
    lam = R.default_phantom(10) + 0.25
    np.testing.assert_array_equal(D.simulate_counts(lam, e, 99), R.simulate_counts(lam, e, 99))


@ref
def test_votes_and_dissimilarity_bitwise():
    import importlib
    R = refload.load()
    cli = importlib.import_module("mmkit_ref.cli")
    votes = D.synthetic_votes(37, 51, 4)
    np.testing.assert_array_equal(votes, cli._synthetic_votes(37, 51, 4))
    np.testing.assert_array_equal(D.votes_to_dissimilarity(votes),
                                  R.votes_to_dissimilarity(votes))


@ref
def test_cbcl_preprocess_bitwise():
    R = refload.load()
    raw = np.random.default_rng(3).random((40, 19)) * 255.0
    np.testing.assert_array_equal(D.cbcl_preprocess(raw), R.cbcl_preprocess(raw))
