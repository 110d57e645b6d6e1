"""Pin the CPU oracle (oracle/port.py) to the real reference's outputs.

Golden vectors come from tests/golden/make_golden.py run against sphdwi 0.1.0.
Tolerances are the reference's own float64 ones (pkg/tests/*: 1e-9 .. 1e-13).
"""

import numpy as np
import pytest

from oracle import port
from conftest import scipy_basis

TWO_SQRT_PI = 2.0 * np.sqrt(np.pi)


@pytest.mark.parametrize("L", [0, 2, 4, 6, 8, 10])
def test_basis_matches_reference(golden, L):
    got = port.eval_basis(golden["basis_dirs"], L)
    assert np.max(np.abs(got - golden[f"basis_o{L}"])) <= 1e-14


@pytest.mark.parametrize("L", [0, 2, 4, 8])
def test_basis_matches_scipy(golden, L):
    # reference KAT: pkg/tests/test_shcore.py:51-56 (atol 1e-13)
    d = golden["basis_dirs"]
    np.testing.assert_allclose(port.eval_basis(d, L), scipy_basis(d, L), atol=1e-13)


def test_basis_kats():
    # pkg/tests/test_shcore.py:39-49, 66-70
    assert abs(port.eval_basis([[0.3, 0.2, 0.9]], 4)[0, 0] - 0.28209479177387814) < 1e-15
    row = port.eval_basis([[0.0, 0.0, 1.0]], 4)[0]
    for j, (l, m) in enumerate([(l, m) for l in (0, 2, 4) for m in range(-l, l + 1)]):
        if m != 0:
            assert row[j] == 0.0
    rng = np.random.default_rng(1)
    d = rng.normal(size=(100, 3))
    assert np.array_equal(port.eval_basis(d, 8), port.eval_basis(-d, 8))


def test_lb_diag(golden):
    assert np.array_equal(port.lb_diag(8), golden["lb_o8"])
    assert np.all(port.lb_diag(4)[1:6] == 36.0) and np.all(port.lb_diag(4)[6:] == 400.0)


@pytest.mark.parametrize("tag,dirs,L,lam", [
    ("d90_o8_l006", "dirs90", 8, 0.006), ("d30_o4_l0", "dirs30", 4, 0.0),
    ("d60_o8_l006", "dirs60", 8, 0.006), ("r40_o6_l06", "fit_r40", 6, 0.06),
    ("d90_o4_l0", "dirs90", 4, 0.0)])
def test_fit_operator(golden, tag, dirs, L, lam):
    M, B, cond = port.fit_operator(golden[dirs], L, lam)
    assert np.max(np.abs(M - golden[f"fit_{tag}"])) <= 1e-12
    assert abs(cond - float(golden[f"cond_{tag}"])) <= 1e-9 * cond


def test_tangent_frames_and_rings(golden):
    for i, u in enumerate(golden["frame_u"]):
        e1, e2 = port.tangent_frame(u)
        assert np.max(np.abs(e1 - golden["frame_e1"][i])) <= 1e-15
        assert np.max(np.abs(e2 - golden["frame_e2"][i])) <= 1e-15
        assert np.max(np.abs(port.ring(u, 0.5, 6) - golden["ring_u_a05_n6"][i])) <= 1e-15
    # pkg/tests/test_shcore.py:150-154
    r = port.ring((0.0, 0.0, 1.0), np.pi / 5, 5)
    np.testing.assert_allclose(r[:, 2], 0.8090169943749475, atol=1e-12)


@pytest.mark.parametrize("tag,args", [
    ("g90", ("dirs90", [5], np.pi / 5, 8, 8, 0.006)),
    ("g30r2", ("dirs30", [4, 8], 0.35, 4, 4, 0.0)),
    ("g30o42", ("dirs30", [5], 0.52, 4, 2, 0.0))])
def test_lsc_geometry(golden, tag, args):
    geo = port.lsc_geometry(golden[args[0]], *args[1:])
    assert np.max(np.abs(geo["resample"] - golden[f"{tag}_resample"])) <= 1e-14
    assert np.max(np.abs(geo["refit"] - golden[f"{tag}_refit"])) <= 1e-12


def test_signal_to_sh(golden):
    M, _, _ = port.fit_operator(golden["dirs90"], 8, 0.006)
    got = port.signal_to_sh(golden["s2sh_x"], M, 3)
    assert np.max(np.abs(got - golden["s2sh_c"])) <= 1e-12


def test_signal_to_sh_per_shell(golden):
    ops = [port.fit_operator(golden["dirs30"], 4, 0.006)[0], port.fit_operator(golden["pershell_dirs_b"], 4, 0.006)[0]]
    got = port.signal_to_sh(golden["pershell_x"], ops, 2)
    assert np.max(np.abs(got - golden["pershell_c"])) <= 1e-12


def test_sh_to_signal(golden):
    for t, key in (("dirs90", "sh2s_y90"), ("sh2s_target60", "sh2s_y60")):
        Bt = port.eval_basis(golden[t], 8)
        got = port.sh_to_signal(golden["sh2s_c"], Bt, 3)
        assert np.max(np.abs(got - golden[key])) <= 1e-12


def test_transform_adjoints(golden):
    M, _, _ = port.fit_operator(golden["dirs90"], 8, 0.006)
    assert np.max(np.abs(port.signal_to_sh_adjoint(golden["s2sh_dc"], M, 3) - golden["s2sh_dx"])) <= 1e-11
    Bt = port.eval_basis(golden["dirs90"], 8)
    assert np.max(np.abs(port.sh_to_signal_adjoint(golden["sh2s_dy"], Bt, 3) - golden["sh2s_dc"])) <= 1e-11


LSC_CASES = [("lsc33", "g90", ("dirs90", [5], np.pi / 5, 8, 8, 0.006)),
             ("lsc32", "g90", ("dirs90", [5], np.pi / 5, 8, 8, 0.006)),
             ("lsc11", "g90", ("dirs90", [5], np.pi / 5, 8, 8, 0.006)),
             ("lscr2", "g30r2", ("dirs30", [4, 8], 0.35, 4, 4, 0.0)),
             ("lsco42", "g30o42", ("dirs30", [5], 0.52, 4, 2, 0.0))]


@pytest.mark.parametrize("tag,gtag,args", LSC_CASES)
def test_lsc_forward_backward(golden, tag, gtag, args):
    geo = port.lsc_geometry(golden[args[0]], *args[1:])
    c, w, b = golden[f"{tag}_c"], golden[f"{tag}_w"], golden[f"{tag}_b"]
    u = port.lsc_forward(c, w, b, geo)
    assert port.rel_err(u, golden[f"{tag}_u"]) <= 1e-12
    dc, dW, db = port.lsc_backward(c, golden[f"{tag}_g"], w, geo)
    assert port.rel_err(dc, golden[f"{tag}_dc"]) <= 1e-12
    assert port.rel_err(dW, golden[f"{tag}_dW"]) <= 1e-12
    assert port.rel_err(db, golden[f"{tag}_db"]) <= 1e-12


def test_chain_forward_backward(golden):
    M, _, _ = port.fit_operator(golden["dirs90"], 8, 0.006)
    geo = port.lsc_geometry(golden["dirs90"], [5], np.pi / 5, 8, 8, 0.006)
    Bt = port.eval_basis(golden["dirs90"], 8)
    x, w, b = golden["s2sh_x"], golden["chain_w"], golden["chain_b"]
    y = port.chain_forward(x, M, geo, w, b, Bt, 3)
    assert port.rel_err(y, golden["chain_y"]) <= 1e-12
    dx, dW, db = port.chain_backward(x, golden["chain_dy"], M, geo, w, Bt, 3)
    assert port.rel_err(dx, golden["chain_dx"]) <= 1e-12
    assert port.rel_err(dW, golden["chain_dW"]) <= 1e-12
    assert port.rel_err(db, golden["chain_db"]) <= 1e-12


def test_constant_signal_kat(golden):
    # pkg/tests/test_fitting.py:72-79: c0 = 2 sqrt(pi) for lambda in {0, .006, .06}
    for lam in (0.0, 0.006, 0.06):
        M, _, _ = port.fit_operator(golden["dirs30"], 4, lam)
        c = port.signal_to_sh(np.ones((1, 30, 2, 1, 1)), M, 1)[0, :, 0, 0, 0]
        assert abs(c[0] - TWO_SQRT_PI) <= 1e-10 and np.max(np.abs(c[1:])) <= 1e-10
