"""Operator-level parity: CUDA path (through the C ABI) vs the C restatement
(oracle/port), which is itself pinned byte-for-byte to the unmodified
reference (tests/test_oracle_port.py). fp64 throughout; tolerances stated per
check (the GPU sums in a different order and uses FMA, so agreement is to
round-off, not bitwise)."""
import numpy as np
import pytest

from paper_1510_07230_b200 import configs

pytestmark = pytest.mark.gpu

SPECS = [
    configs.small_molecule(16, 4, L=8.0),
    configs.ProblemSpec("skew", (12, 10, 14), (7.0, 6.0, 9.0),
                        [(3.0, 2.5, 4.0, 3.0, 1.0), (4.5, 3.2, 5.5, 1.0, 0.7)], 5),
]


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


@pytest.fixture(params=SPECS, ids=[s.name for s in SPECS])
def setup(request, port, native):
    spec = request.param
    u0 = port.random_orthonormal(spec)
    e = native.engine_for(spec)
    yield spec, u0, e
    e.close()


def test_random_block_bits(port, native):
    spec = SPECS[1]
    e = native.engine_for(spec)
    b = e.alloc()
    e.random_block(b, 42)
    got = e.download(b)
    want = port.random_normals(42, spec.n_orbitals * spec.num_points).reshape(spec.n_orbitals, -1)
    assert np.array_equal(got, want)  # same generator, same bits (rng.hpp:13-41)
    e.close()


def test_external_potential(setup, port, native):
    spec, _, e = setup
    got = e.get_field(native.PO_VEXT)
    assert rel(got, port.external_potential(spec)) < 1e-14


def test_laplacian(setup, port, native):
    spec, u0, e = setup
    u = e.block_from(u0)
    out = e.alloc()
    e.laplacian(u, out)
    got = e.download(out)
    want = np.stack([port.laplacian(spec, x) for x in u0])
    assert rel(got, want) < 1e-13


def test_build_hamiltonian_and_apply(setup, port, native):
    spec, u0, e = setup
    e.set_poisson_solver("cg")  # the reference's algorithm: iteration counts comparable
    u = e.block_from(u0)
    eh, exc, iters = e.build_hamiltonian(u, True, True)
    st = port.build_hamiltonian(spec, u0)
    assert rel(e.get_field(native.PO_RHO), st["rho"]) < 1e-14
    assert rel(e.get_field(native.PO_VXC), st["v_xc"]) < 1e-13
    # both CG solves stop at ||r|| <= 1e-10 ||b|| (energy.cpp:105-143)
    assert rel(e.get_field(native.PO_VH), st["v_h"]) < 1e-8
    assert rel(e.get_field(native.PO_VLOCAL), st["v_local"]) < 1e-8
    assert iters > 0 and abs(iters - st["cg_iters"]) <= max(3, st["cg_iters"] // 10)
    en, kin, ext = port.total_energy(spec, u0, st)
    assert abs(eh - en["hartree"]) < 1e-9 * max(1.0, abs(en["hartree"]))
    assert abs(exc - en["xc"]) < 1e-12 * max(1.0, abs(en["xc"]))
    hu = e.alloc()
    sig, k, x = e.apply_hamiltonian(u, hu)
    want_hu = port.apply_hamiltonian(spec, e.get_field(native.PO_VLOCAL), u0)
    assert rel(e.download(hu), want_hu) < 1e-12
    assert np.allclose(k, kin, rtol=1e-11, atol=1e-12)
    assert np.allclose(x, ext, rtol=1e-11, atol=1e-12)
    wq = np.prod(spec.spacing)
    assert np.allclose(sig, wq * np.einsum("ip,ip->i", want_hu, u0), rtol=1e-10, atol=1e-12)
    tot = e.total_energy(u)
    assert abs(tot["total"] - en["total"]) < 1e-8


@pytest.mark.parametrize("mode", ["cg", "cg_warm", "dst"])
def test_poisson_modes(setup, port, native, mode):
    """Every Poisson mode stops on the reference's criterion ||b - A x|| <=
    1e-10 ||b|| (energy.cpp:120-142); the DST start makes CG converge at once."""
    spec, u0, e = setup
    e.set_poisson_solver(mode)
    u = e.block_from(u0)
    eh, _, iters = e.build_hamiltonian(u, True, True)
    st = port.build_hamiltonian(spec, u0)
    assert rel(e.get_field(native.PO_VH), st["v_h"]) < 1e-8
    en, _, _ = port.total_energy(spec, u0, st)
    assert abs(eh - en["hartree"]) < 1e-9 * max(1.0, abs(en["hartree"]))
    if mode == "dst":
        assert iters <= 2
    else:
        assert iters > 0


@pytest.mark.parametrize("n", [(15, 12, 10), (9, 7, 13)])  # even / odd plane sizes
def test_poisson_closed_form(native, n):
    """KAT after test_energy.cpp:229-286: rho = sin-mode product has the exact
    discrete solution v = 4 pi rho / lambda (relative error <= 1e-8)."""
    L = (6.0, 5.0, 4.0)
    spec = configs.ProblemSpec("kat", n, L, [], 1)
    e = native.engine_for(spec)
    h = [L[a] / (n[a] + 1) for a in range(3)]
    modes = (1, 2, 3)
    k = [np.arange(1, n[a] + 1) for a in range(3)]
    s = [np.sin(np.pi * modes[a] * k[a] / (n[a] + 1)) for a in range(3)]
    u = np.einsum("i,j,k->ijk", s[0], s[1], s[2]).reshape(1, -1)
    lam = sum(4.0 * np.sin(np.pi * modes[a] / (2 * (n[a] + 1))) ** 2 / h[a] ** 2 for a in range(3))
    rho = u[0] ** 2
    for mode in ("cg", "dst"):
        e.set_poisson_solver(mode)
        # density of a single orbital u is u^2; solve with that rho via a 1-orbital block
        b = e.block_from(u)
        e.build_hamiltonian(b, True, False)
        vh = e.get_field(native.PO_VH)
        # -lap vh = 4 pi rho  <=>  check residual with the port-independent DST in numpy
        from numpy.fft import fft  # noqa: F401 (kept simple: verify via residual)
        lap = np.zeros_like(vh).reshape(n)
        v3 = vh.reshape(n)
        for a in range(3):
            sl = [slice(None)] * 3
            vp = np.zeros_like(v3)
            vm = np.zeros_like(v3)
            idx_p = [slice(None)] * 3
            idx_p[a] = slice(0, n[a] - 1)
            src_p = [slice(None)] * 3
            src_p[a] = slice(1, n[a])
            vp[tuple(idx_p)] = v3[tuple(src_p)]
            vm[tuple(src_p)] = v3[tuple(idx_p)]
            lap += (vm - 2 * v3 + vp) / h[a] ** 2
            del sl
        res = -lap.ravel() - 4 * np.pi * rho
        assert np.linalg.norm(res) <= 1e-10 * np.linalg.norm(4 * np.pi * rho) * 1.0001
    # sin-mode Laplacian eigenvalue sanity (grid.cpp stencil, test_grid.cpp:74-91)
    out = e.alloc()
    e.laplacian(e.block_from(u), out)
    assert rel(e.download(out), -lam * u) < 1e-12
    e.close()


def test_gram_mix(setup, port, native):
    spec, u0, e = setup
    rng = np.random.default_rng(3)
    a = rng.standard_normal(u0.shape)
    ba, bu = e.block_from(a), e.block_from(u0)
    g_sym = e.gram(ba, ba)
    assert np.array_equal(g_sym, g_sym.T)  # exact symmetric fill (manifold.cpp:45-53)
    assert rel(g_sym, port.gram(spec, a, a, same=True)) < 1e-13
    assert rel(e.gram(ba, bu), port.gram(spec, a, u0)) < 1e-12
    m = rng.standard_normal((spec.n_orbitals, spec.n_orbitals))
    out = e.alloc()
    e.mix(ba, m, out)
    assert rel(e.download(out), m.T @ a) < 1e-13


@pytest.mark.parametrize("n_orb", [1, 8, 9, 13, 17, 33, 34, 42, 56, 64])
def test_dmma_small_n(native, n_orb):
    """Register-resident small-N Gram / mix paths (N <= 64), incl. the
    triangular-skip rotation used for U L^{-T}."""
    spec = configs.ProblemSpec("smalln", (10, 9, 11), (5.0, 5.0, 5.0), [], n_orb, hartree=False, xc=False)
    e = native.engine_for(spec)
    rng = np.random.default_rng(100 + n_orb)
    a = rng.standard_normal((n_orb, spec.num_points))
    b = rng.standard_normal((n_orb, spec.num_points))
    ba, bb = e.block_from(a), e.block_from(b)
    wq = np.prod(spec.spacing)
    g = e.gram(ba, ba)
    assert np.array_equal(g, g.T)
    assert rel(g, wq * a @ a.T) < 1e-12
    assert rel(e.gram(ba, bb), wq * a @ b.T) < 1e-12
    out = e.alloc()
    m = rng.standard_normal((n_orb, n_orb))
    e.mix(ba, m, out)
    assert rel(e.download(out), m.T @ a) < 1e-12
    # orthonormalize exercises the upper-triangular (L^{-T}) skip path
    pre, dev, fb = e.orthonormalize(ba, out, True)
    w = e.download(out)
    assert np.abs(wq * w @ w.T - np.eye(n_orb)).max() < 1e-12
    e.close()


@pytest.mark.parametrize("n_orb,n", [(49, (9, 8, 10)), (67, (9, 8, 10)), (130, (9, 8, 10)),
                                     (200, (24, 20, 22)), (300, (12, 13, 14))])
def test_dmma_multitile(port, native, n_orb, n):
    """N > 48 exercises the tiled TMA Gram (64- and 128-wide tiles, upper-only
    in the symmetric path, diagonal tiles skipping the lower fragments) and
    several mix orbital tiles."""
    spec = configs.ProblemSpec("tile", n, (5.0, 5.0, 5.0), [], n_orb, hartree=False, xc=False)
    e = native.engine_for(spec)
    rng = np.random.default_rng(n_orb)
    a = rng.standard_normal((n_orb, spec.num_points))
    b = rng.standard_normal((n_orb, spec.num_points))
    ba, bb = e.block_from(a), e.block_from(b)
    wq = np.prod(spec.spacing)
    g = e.gram(ba, ba)
    assert np.array_equal(g, g.T)
    assert rel(g, wq * a @ a.T) < 1e-12
    assert rel(e.gram(ba, bb), wq * a @ b.T) < 1e-12
    m = rng.standard_normal((n_orb, n_orb))
    out = e.alloc()
    e.mix(ba, m, out)
    assert rel(e.download(out), m.T @ a) < 1e-12
    e.close()


@pytest.mark.parametrize("n_orb,n", [(65, (9, 9, 11)), (67, (9, 9, 11)), (128, (12, 13, 14)),
                                     (130, (9, 9, 11)), (200, (24, 20, 22)), (256, (10, 9, 11)),
                                     (260, (10, 9, 11))])
def test_mix_big(native, n_orb, n):
    """Large-N TMA mix (N > 64, manifold.cpp:67-85): full, upper-triangular
    (L^{-T}, manifold.cpp:97-114), the trial rotation (W - tau Z) L^{-T} and the
    gradient norms of D = HW - W Sigma (manifold.cpp:181-202); odd point counts
    exercise the ragged last tile, N > 128 several orbital tiles; N = 128 / 256 take
    the balanced triangular kernel (forward / backward point halves)."""
    spec = configs.ProblemSpec("mixbig", n, (5.0, 5.0, 5.0), [], n_orb, hartree=False, xc=False)
    e = native.engine_for(spec)
    rng = np.random.default_rng(11 + n_orb)
    a = rng.standard_normal((n_orb, spec.num_points))
    b = rng.standard_normal((n_orb, spec.num_points))
    ba, bb, out = e.block_from(a), e.block_from(b), e.alloc()
    m = rng.standard_normal((n_orb, n_orb))
    e.mix(ba, m, out)
    assert rel(e.download(out), m.T @ a) < 1e-12
    mu = np.triu(m)
    e.set_matrix(mu)
    e.enqueue("mix_upper", a=ba, out=out)
    assert rel(e.download(out), mu.T @ a) < 1e-12
    e.enqueue("rotation", a=ba, b=bb, out=out)
    assert rel(e.download(out), mu.T @ (a - 0.3 * b)) < 1e-12
    # orthonormalisation: Cholesky + L^{-T} on the device, then the triangular mix
    wq = np.prod(spec.spacing)
    pre, dev, fb = e.orthonormalize(ba, out, True)
    assert not fb and 0.0 <= dev <= 1e-12
    wo = e.download(out)
    assert np.abs(wq * wo @ wo.T - np.eye(n_orb)).max() < 1e-12
    l_ref = np.linalg.cholesky(wq * a @ a.T)
    assert rel(wo, np.linalg.solve(l_ref, a)) < 1e-9
    # ||HW - W Sigma||^2 per orbital on an orthonormal W with HW = S W (S symmetric)
    q, _ = np.linalg.qr(a.T)
    w = q.T / np.sqrt(wq)
    s = rng.standard_normal((n_orb, n_orb))
    s = s + s.T
    hw = s @ w + 1e-3 * rng.standard_normal(w.shape)
    hw = hw - 0.5 * ((hw @ w.T) * wq - (w @ hw.T) * wq) @ w  # keep <HW, W> symmetric
    sig, dd = e.stiefel_gradient(e.block_from(w), e.block_from(hw))
    d_ref = hw - sig.T @ w
    assert np.allclose(dd, wq * np.einsum("ip,ip->i", d_ref, d_ref), rtol=1e-9, atol=1e-14)
    e.close()


def test_orthonormalize(setup, port, native):
    spec, u0, e = setup
    rng = np.random.default_rng(5)
    trial = u0 + 0.3 * rng.standard_normal(u0.shape)
    bt, bo = e.block_from(trial), e.alloc()
    pre, dev, fb = e.orthonormalize(bt, bo, True)
    w_ref, pre_ref, dev_ref, fb_ref = port.orthonormalize(spec, trial)
    assert not fb and not fb_ref
    assert rel(pre, pre_ref) < 1e-13
    assert rel(e.download(bo), w_ref) < 1e-10
    assert 0.0 <= dev <= 1e-12 and dev_ref <= 1e-12


def test_orthonormalize_degenerate(native):
    spec = configs.small_molecule(8, 3, L=6.0)
    e = native.engine_for(spec)
    a = np.ones((3, spec.num_points))
    with pytest.raises(native.DegenerateSetError):
        e.orthonormalize(e.block_from(a), e.alloc(), True)
    e.close()


def test_residuals_gradient_rotation(setup, port, native):
    spec, u0, e = setup
    u = e.block_from(u0)
    e.build_hamiltonian(u)
    hu = e.alloc()
    e.apply_hamiltonian(u, hu)
    hu_h = e.download(hu)
    z = e.alloc()
    sig, zz = e.diagonal_residuals(u, hu, z)
    wq = np.prod(spec.spacing)
    s_ref = wq * np.einsum("ip,ip->i", hu_h, u0)
    z_ref = hu_h - s_ref[:, None] * u0
    assert np.allclose(sig, s_ref, rtol=1e-12, atol=1e-13)
    assert rel(e.download(z), z_ref) < 1e-11
    assert np.allclose(zz, wq * np.einsum("ip,ip->i", z_ref, z_ref), rtol=1e-10)
    sigma, dd = e.stiefel_gradient(u, hu)
    sigma_ref = port.gram(spec, hu_h, u0)
    assert rel(sigma, sigma_ref) < 1e-12
    d_ref = hu_h - sigma_ref.T @ u0
    assert np.allclose(dd, wq * np.einsum("ip,ip->i", d_ref, d_ref), rtol=1e-9, atol=1e-14)
    gam, p = e.subspace_rotate(u, 0.5 * (sigma + sigma.T))
    gam_ref, p_ref = port.subspace_rotate(0.5 * (sigma + sigma.T))
    assert np.allclose(gam, gam_ref, atol=1e-11)
    assert np.allclose(p, p_ref, atol=1e-8)  # sign rule, manifold.cpp:233-241
    assert rel(e.download(u), p_ref.T @ u0) < 1e-8


def test_bb_products_and_lincomb(setup, native):
    spec, u0, e = setup
    rng = np.random.default_rng(9)
    blocks = [rng.standard_normal(u0.shape) for _ in range(4)]
    h = [e.block_from(x) for x in blocks]
    ss, sy, yy = e.bb_products(*h)
    wq = np.prod(spec.spacing)
    s = blocks[0] - blocks[1]
    y = blocks[2] - blocks[3]
    assert np.allclose(ss, wq * (s * s).sum(1), rtol=1e-12)
    assert np.allclose(sy, wq * (s * y).sum(1), rtol=1e-10, atol=1e-12)
    assert np.allclose(yy, wq * (y * y).sum(1), rtol=1e-12)
    out = e.alloc()
    e.linear_combination(h[0], -0.25, h[1], out)
    assert rel(e.download(out), blocks[0] - 0.25 * blocks[1]) < 1e-15


def test_invalid_arguments(native):
    with pytest.raises(native.InvalidArgument):
        native.Engine((0, 4, 4), (1.0, 1.0, 1.0), 2)
    with pytest.raises(native.InvalidArgument):
        native.Engine((4, 4, 4), (1.0, -1.0, 1.0), 2)
    with pytest.raises(native.InvalidArgument):
        native.Engine((2, 2, 2), (1.0, 1.0, 1.0), 9)  # more orbitals than points
    e = native.Engine((4, 4, 4), (4.0, 4.0, 4.0), 2)
    with pytest.raises(native.InvalidArgument):
        e.external_potential([(9.0, 1.0, 1.0, 1.0, 1.0)])  # outside the box (energy.cpp:20-30)
    with pytest.raises(native.InvalidArgument):
        e.download(17)  # bad handle
    e.close()


@pytest.mark.parametrize("n_orb", [1, 4, 5, 9, 13, 17, 33, 34, 48, 67, 200, 260])
def test_gram_fused_trial(native, n_orb):
    """Gram of W - tau Z formed inside the load (optimizer.cpp:459-463)."""
    spec = configs.ProblemSpec("trial", (10, 9, 11), (5.0, 5.0, 5.0), [], n_orb, hartree=False, xc=False)
    e = native.engine_for(spec)
    rng = np.random.default_rng(7 + n_orb)
    w = rng.standard_normal((n_orb, spec.num_points))
    z = rng.standard_normal((n_orb, spec.num_points))
    bw, bz = e.block_from(w), e.block_from(z)
    t = w - 0.37 * z
    wq = np.prod(spec.spacing)
    g = e.gram_lincomb(bw, -0.37, bz)
    assert np.array_equal(g, g.T)
    assert rel(g, wq * t @ t.T) < 1e-12
    e.close()


@pytest.mark.parametrize("n_orb,hist", [(128, True), (128, False), (80, True), (65, True), (33, True), (130, True),
                                        (260, True)])
def test_direction_sums(native, n_orb, hist):
    """po_direction_sums — the iteration's direction step with z implicit
    (optimizer.cpp:265-320, 386-397; manifold.cpp:183, 204-216): sigma_ii,
    Sigma = <(HU)^T U>, ||z_i||^2 and the BB products against (u_prev, z_prev =
    hu_prev - sigma_prev u_prev), vs the same formulas in numpy fp64. N > 64 takes
    the one-pass form (the Sigma Gram's DMMA warps carry the sums; N = 130 / 260:
    several 128-tiles, the sums on the diagonal ones), N = 33 the Gram + a
    streaming pass. Sums of ~2700 terms in another order: 1e-12 relative."""
    # N = 65: an odd point count too (13 x 11 x 15: the last 16-point stage is ragged)
    spec = (configs.ProblemSpec("odd", (13, 11, 15), (7.0, 6.0, 9.0), [(3.0, 2.5, 4.0, 3.0, 1.0)], n_orb)
            if n_orb == 65 else configs.small_molecule(14, n_orb, L=8.0))
    rng = np.random.default_rng(5)
    wq = float(np.prod(spec.spacing))
    u = rng.standard_normal((n_orb, spec.num_points))
    hu = 0.7 * u + 0.3 * rng.standard_normal(u.shape)
    up = u + 0.05 * rng.standard_normal(u.shape)
    hup = hu + 0.05 * rng.standard_normal(u.shape)
    e = native.engine_for(spec)
    bu, bhu = e.block_from(u), e.block_from(hu)
    sig = wq * np.einsum("ip,ip->i", hu, u)
    z = hu - sig[:, None] * u
    want = dict(sigma_diag=sig, sigma=wq * hu @ u.T, zz=wq * np.einsum("ip,ip->i", z, z))
    if hist:
        bup, bhup = e.block_from(up), e.block_from(hup)
        sigp = wq * np.einsum("ip,ip->i", hup, up)
        zp = hup - sigp[:, None] * up
        s, y = u - up, z - zp
        want.update(ss=wq * np.einsum("ip,ip->i", s, s), sy=wq * np.einsum("ip,ip->i", s, y),
                    yy=wq * np.einsum("ip,ip->i", y, y))
        got = e.direction_sums(bu, bhu, bup, bhup, sigp)
    else:
        got = e.direction_sums(bu, bhu)
    assert set(got) == set(want)
    for k, v in want.items():
        assert rel(got[k], v) < 1e-12, k
    e.close()
