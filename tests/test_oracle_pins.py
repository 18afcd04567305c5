"""Oracle vs values printed in SPEC.md / derived by hand (tests/golden/spec_examples.json)."""
import numpy as np
import pytest

import oracle
from oracle import lcae_oracle as O


def _field(ex, **over):
    d = dict(ex)
    d.update(over)
    return O.rica_field(np.array(d["W"], float), d["alpha"], np.array(d["b"], float),
                        np.array(d["x"], float), d["lam"], d["eps"], d.get("g", 1))


def test_worked_example_objective(golden):
    ex = golden["objective_worked_example"]
    o = _field(ex)
    assert o["J_rec"] == pytest.approx(ex["J_rec"], abs=1e-15)
    assert o["J_sparse"] == pytest.approx(ex["J_sparse"], abs=1e-15)
    assert o["J_rec"] + o["J_sparse"] == pytest.approx(ex["J"], abs=1e-15)
    assert O.rica_objective(np.array(ex["W"], float), ex["alpha"], np.array(ex["b"], float),
                            np.array(ex["x"], float), ex["lam"], ex["eps"]) == pytest.approx(2.4, abs=1e-15)


def test_worked_example_gradients(golden):
    ex = golden["objective_worked_example"]
    gr = golden["objective_worked_example_gradients"]
    o = _field(ex)
    np.testing.assert_allclose(o["dW"], gr["dW"], atol=1e-14)
    assert o["dalpha"] == pytest.approx(gr["dalpha"], abs=1e-14)
    np.testing.assert_allclose(o["db"], gr["db"], atol=1e-14)
    np.testing.assert_allclose(o["dx"], gr["dx"], atol=1e-14)


def test_worked_example_pool2(golden):
    ex = golden["objective_worked_example"]
    gp = golden["objective_worked_example_pool2"]
    o = _field(ex, g=2)
    assert o["J_rec"] + o["J_sparse"] == pytest.approx(gp["J"], abs=1e-14)
    np.testing.assert_allclose(o["dW"], gp["dW"], atol=1e-13)
    assert o["dalpha"] == pytest.approx(gp["dalpha"], abs=1e-13)
    np.testing.assert_allclose(o["db"], gp["db"], atol=1e-14)
    np.testing.assert_allclose(o["dx"], gp["dx"], atol=1e-13)


def test_zero_input_objective(golden):
    o = O.rica_field(np.eye(3, 5), 1.3, np.zeros(5), np.zeros((4, 5)), 0.1, 0.0, 1)
    assert o["J_rec"] + o["J_sparse"] == golden["objective_zero_input"]["J"]
    assert np.all(o["dW"] == 0) and o["dalpha"] == 0 and np.all(o["db"] == 0) and np.all(o["dx"] == 0)


def test_db_example(golden):
    ex = golden["db_example"]
    o = _field(ex)
    np.testing.assert_allclose(o["db"], ex["db"], atol=1e-14)


def test_geometry_examples(golden):
    for cs in golden["geometry"]["cases"]:
        (H, W, C), (fh, fw), s = cs["img"], cs["rf"], cs["stride"]
        gr, gc = O.field_grid(H, W, fh, fw, s)
        assert [gr, gc] == cs["grid"] and gr * gc == cs["fields"]
    for cs in golden["geometry"]["errors"]:
        (H, W, C), (fh, fw), s = cs["img"], cs["rf"], cs["stride"]
        with pytest.raises(O.GeometryError, match=f"residue rows={cs['residue']}"):
            O.field_grid(H, W, fh, fw, s)
    with pytest.raises(O.GeometryError):
        O.field_grid(8, 8, 9, 4, 1)


def test_param_count(golden):
    for cs in golden["param_count"]["cases"]:
        assert O.param_count(cs["fields"], cs["k"], cs["n"]) == cs["total"]


def test_projection_examples(golden):
    for cs in golden["projection"]["cases"]:
        np.testing.assert_allclose(O.project_row_norms(np.array([cs["row"]], float))[0], cs["out"], atol=1e-16)
    with pytest.raises(O.DegenerateRowError):
        O.project_row_norms(np.array([golden["projection"]["degenerate"]], float))
    rng = np.random.default_rng(3)
    W = rng.standard_normal((5, 7))
    P1 = O.project_row_norms(W)
    np.testing.assert_allclose(O.project_row_norms(P1), P1, rtol=0, atol=2e-16)  # idempotent


def test_sgd_examples(golden):
    ex = golden["sgd"]
    W = O.project_row_norms(np.random.default_rng(0).standard_normal((1, 3, 4)))
    grads = dict(dW=np.zeros_like(W), dalpha=np.array([ex["dalpha"]]), db=np.zeros((1, 4)))
    Wn, an, bn, _, nre = O.sgd_update(W, np.array([ex["alpha"]]), np.zeros((1, 4)), grads, ex["lr"])
    assert an[0] == pytest.approx(ex["alpha_after"], abs=1e-15)
    np.testing.assert_allclose(Wn, W, atol=1e-15)  # zero W-gradient: projection is a no-op
    assert nre == 0
    # alpha clamp
    _, an, _, _, _ = O.sgd_update(W, np.array([0.05]), np.zeros((1, 4)), grads, 0.1, alpha_min=1e-8)
    assert an[0] == 1e-8


def test_degenerate_row_reinit():
    W = np.zeros((2, 3, 6))
    W[:, :, 0] = 1.0
    grads = dict(dW=np.zeros_like(W), dalpha=np.zeros(2), db=np.zeros((2, 6)))
    grads["dW"][1, 2, 0] = 10.0     # lr*dW cancels row (1,2) exactly -> degenerate
    Wn, _, _, _, nre = O.sgd_update(W, np.ones(2), np.zeros((2, 6)), grads, 0.1, seed=5, step=3)
    assert nre == 1
    np.testing.assert_allclose(np.linalg.norm(Wn, axis=-1), 1.0, atol=1e-15)
    np.testing.assert_allclose(Wn[1, 2], O.reinit_row(5, 3, 1, 2, 6), atol=0)
    assert not np.allclose(O.reinit_row(5, 3, 1, 2, 6), O.reinit_row(5, 4, 1, 2, 6))


def test_splitmix64_reference_values():
    # SplitMix64 published test vector: seed 0 -> first output 0xE220A8397B1DCDAF
    assert O.splitmix64(0) == 0xE220A8397B1DCDAF
