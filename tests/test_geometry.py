"""Host-side float64 builders (paper_1808_01517_b200/geometry.py) vs the reference's golden vectors
and the reference tests' known answers (pkg/tests/test_shcore.py, test_fitting.py, test_lsc.py)."""

import numpy as np
import pytest

import paper_1808_01517_b200 as dl
from paper_1808_01517_b200 import geometry as geo
from paper_1808_01517_b200.directions import unit_sphere_directions
from conftest import random_unit_vectors, scipy_basis

TWO_SQRT_PI = 2.0 * np.sqrt(np.pi)


def test_direction_tables_match_reference(golden):
    for n in (30, 60, 90):
        assert np.array_equal(unit_sphere_directions(n), golden[f"dirs{n}"])
    with pytest.raises(ValueError):
        unit_sphere_directions(45)


class TestPacking:
    def test_index_kats(self):
        assert geo.sh_index(0, 0) == 0 and geo.sh_index(2, -2) == 1 and geo.sh_index(4, 4) == 14
        assert [geo.coeff_count(o) for o in (0, 2, 4, 6, 8)] == [1, 6, 15, 28, 45]

    def test_round_trip(self):
        for l in range(0, 13, 2):
            for m in range(-l, l + 1):
                assert geo.sh_degree_order(geo.sh_index(l, m)) == (l, m)

    @pytest.mark.parametrize("l,m", [(1, 0), (3, 2), (-2, 0), (2, 3), (4, -5)])
    def test_invalid(self, l, m):
        with pytest.raises(ValueError):
            geo.sh_index(l, m)

    @pytest.mark.parametrize("order", [-2, 3, 7])
    def test_bad_order(self, order):
        with pytest.raises(ValueError):
            geo.coeff_count(order)


class TestBasis:
    @pytest.mark.parametrize("L", [0, 2, 4, 6, 8, 10])
    def test_matches_reference(self, golden, L):
        assert np.max(np.abs(geo.eval_basis(golden["basis_dirs"], L) - golden[f"basis_o{L}"])) <= 1e-14

    def test_scipy_oracle(self, rng):
        d = random_unit_vectors(rng, 300)
        for L in (0, 2, 4, 8):
            np.testing.assert_allclose(geo.eval_basis(d, L), scipy_basis(d, L), atol=1e-13)

    def test_pole_and_parity(self, rng):
        row = geo.eval_basis([[0.0, 0.0, 1.0]], 4)[0]
        for l in (2, 4):
            for m in range(-l, l + 1):
                if m:
                    assert row[geo.sh_index(l, m)] == 0.0
        d = random_unit_vectors(rng, 500)
        assert np.array_equal(geo.eval_basis(d, 8), geo.eval_basis(-d, 8))

    def test_addition_theorem(self, rng):
        b = geo.eval_basis(random_unit_vectors(rng, 50), 8)
        for l in (0, 2, 4, 6, 8):
            idx = [geo.sh_index(l, m) for m in range(-l, l + 1)]
            np.testing.assert_allclose(np.sum(b[:, idx] ** 2, axis=1), (2 * l + 1) / (4 * np.pi), atol=1e-10)

    def test_rejections(self):
        with pytest.raises(ValueError):
            geo.eval_basis(np.empty((0, 3)), 4)
        with pytest.raises(ValueError):
            geo.eval_basis([[0, 0, 1]], 3)
        with pytest.raises(ValueError, match="zero direction"):
            geo.as_unit_directions([[0.0, 0.0, 0.0]])
        with pytest.raises(ValueError):
            geo.as_unit_directions([[np.nan, 0, 1]])

    def test_lb(self, golden):
        assert np.array_equal(geo.laplace_beltrami_diag(8), golden["lb_o8"])


class TestFitOperator:
    @pytest.mark.parametrize("tag,dirs,L,lam", [
        ("d90_o8_l006", "dirs90", 8, 0.006), ("d30_o4_l0", "dirs30", 4, 0.0),
        ("d60_o8_l006", "dirs60", 8, 0.006), ("r40_o6_l06", "fit_r40", 6, 0.06), ("d90_o4_l0", "dirs90", 4, 0.0)])
    def test_matches_reference(self, golden, tag, dirs, L, lam):
        op = geo.make_fit_operator(golden[dirs], L, lam)
        assert np.max(np.abs(op.fit_matrix - golden[f"fit_{tag}"])) <= 1e-12
        assert op.cond == pytest.approx(float(golden[f"cond_{tag}"]), rel=1e-9)

    def test_pseudo_inverse(self):
        op = geo.make_fit_operator(unit_sphere_directions(30), 4, 0.0)
        np.testing.assert_allclose(op.fit_matrix @ op.basis_matrix, np.eye(15), atol=1e-9)

    def test_errors(self):
        d = unit_sphere_directions(30)
        with pytest.raises(dl.IllPosedFitError, match="R = 15"):
            geo.make_fit_operator(d[:6], 4, 0.0)
        with pytest.raises(dl.IllPosedFitError, match="cond"):
            geo.make_fit_operator(np.tile([[0.0, 0.0, 1.0]], (20, 1)), 4, 0.0)
        with pytest.raises(ValueError):
            geo.make_fit_operator(d, 4, -1.0)

    def test_read_only(self):
        op = geo.make_fit_operator(unit_sphere_directions(30), 4, 0.006)
        for a in (op.fit_matrix, op.basis_matrix, op.gradients):
            with pytest.raises(ValueError):
                a[0, 0] = 1.0

    @pytest.mark.parametrize("lam", [0.0, 0.006, 0.06])
    def test_constant_signal_kat(self, lam):
        M = geo.make_fit_operator(unit_sphere_directions(30), 4, lam).fit_matrix
        c = M @ np.ones(30)
        assert abs(c[0] - TWO_SQRT_PI) <= 1e-10 and np.max(np.abs(c[1:])) <= 1e-10


class TestRingsAndGeometry:
    def test_frames_and_rings(self, golden):
        for i, u in enumerate(golden["frame_u"]):
            e1, e2 = geo.tangent_basis(u)
            assert np.max(np.abs(e1 - golden["frame_e1"][i])) <= 1e-15
            assert np.max(np.abs(e2 - golden["frame_e2"][i])) <= 1e-15
            assert np.max(np.abs(geo.ring_directions(u, 0.5, 6) - golden["ring_u_a05_n6"][i])) <= 1e-15

    def test_ring_kat(self):
        r = geo.ring_directions((0.0, 0.0, 1.0), np.pi / 5, 5)
        np.testing.assert_allclose(r[:, 2], 0.8090169943749475, atol=1e-12)

    @pytest.mark.parametrize("alpha", [0.0, -0.1, np.pi / 2, 2.0])
    def test_alpha_range(self, alpha):
        with pytest.raises(ValueError):
            geo.ring_directions((0, 0, 1), alpha, 5)

    @pytest.mark.parametrize("tag,args", [
        ("g90", ("dirs90", [5], np.pi / 5, 8, 8, 0.006)),
        ("g30r2", ("dirs30", [4, 8], 0.35, 4, 4, 0.0)),
        ("g30o42", ("dirs30", [5], 0.52, 4, 2, 0.0))])
    def test_geometry_matches_reference(self, golden, tag, args):
        g = geo.build_lsc_geometry(golden[args[0]], *args[1:])
        assert np.max(np.abs(g.resample_matrix - golden[f"{tag}_resample"])) <= 1e-14
        assert np.max(np.abs(g.refit.fit_matrix - golden[f"{tag}_refit"])) <= 1e-12
        assert g.kernel_len == 1 + sum(args[1])

    def test_fold_identity(self, golden):
        # P_k = F Rs[k::K], beta = F 1 = 2 sqrt(pi) e0 (Lambda_00 = 0)
        g = geo.build_lsc_geometry(golden["dirs90"], [5], np.pi / 5, 8, 8, 0.006)
        F, Rs = g.refit.fit_matrix, g.resample_matrix
        for k in range(6):
            assert np.max(np.abs(g.fold[k] - F @ Rs[k::6])) <= 1e-13
        e0 = np.zeros(45)
        e0[0] = TWO_SQRT_PI
        assert np.max(np.abs(g.beta - e0)) <= 1e-12

    def test_hemisphere_and_sizes(self):
        d = unit_sphere_directions(30)
        with pytest.raises(ValueError, match="hemisphere"):
            geo.build_lsc_geometry(d, [5, 5, 5], 0.6, 4, 4, 0.0)
        with pytest.raises(ValueError):
            geo.build_lsc_geometry(d, [], 0.3, 4, 4, 0.0)

    def test_kernels(self):
        k = geo.make_moving_average_kernel([5], shells_in=2, shells_out=1)
        assert k.weights.shape == (1, 2, 6) and np.all(k.weights == 1.0 / 12.0)
        i = geo.make_identity_kernel([5], shells=2)
        assert i.weights[0, 0, 0] == 1 and i.weights[1, 1, 0] == 1 and i.weights.sum() == 2
        with pytest.raises(dl.ShapeError):
            geo.LscKernel(weights=np.full((1, 1, 3), np.nan), bias=np.zeros(1))


def test_modules_construct_on_cpu():
    d = unit_sphere_directions(90)
    lsc = dl.LocalSphericalConvolution(3, 2, 8, 6, d, [5], lb_lambda=0.006, angular_distance=np.pi / 5)
    assert tuple(lsc.sconv.weight.shape) == (2, 3, 1, 6) and tuple(lsc.sconv.bias.shape) == (2,)
    assert tuple(lsc.fold.shape) == (6, 28, 45)
    assert set(lsc.state_dict()) == {"sconv.weight", "sconv.bias"}
    s2 = dl.Signal2SH(8, np.stack([d, d[::-1]]), lb_lambda=0.006)
    assert s2.per_shell and s2.shells == 2 and tuple(s2.fit_matrix.shape) == (2, 45, 90)
    k = lsc.kernel
    lsc.load_kernel(k)
    with pytest.raises(dl.KernelMismatchError):
        lsc.load_kernel(geo.LscKernel(np.zeros((2, 3, 4)), np.zeros(2)))
