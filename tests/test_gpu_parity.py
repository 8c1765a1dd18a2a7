"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.

Bars (BASELINE.json north_star): relative l2 <= 1e-12 for ComplexF64 and
<= 2e-5 for ComplexF32; the node binning / sort permutation bit-exact.
"""

import numpy as np
import pytest

from conftest import rel_l2
from oracle import binning as obin
from oracle import nfft as onfft
from oracle import window as owin
from paper_2208_00049_b200 import workloads

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-12, "c64": 2e-5}


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


# first-generation tile-mode variants: compiled only with -DNFFTB_TILE_VARIANTS
VARIANTS = ("tiled_cas", "tiled_loc", "tiled_own", "tiled_sorted", "tiled_v1")


def _plan(w, **kw):
    torch = _torch()
    import paper_2208_00049_b200 as pkg
    nodes = torch.from_numpy(np.ascontiguousarray(w["nodes"])).cuda()
    try:
        plan = pkg.NfftPlan(nodes, w["N"], m=w["m"], sigma=w["sigma"], precision=w["precision"],
                            batch=w["batch"], **kw)
    except pkg.NfftError as e:
        if kw.get("method") in VARIANTS and e.name == "NFFT_ERROR_UNSUPPORTED":
            pytest.skip(f"{kw['method']} not built (reference variant, -DNFFTB_TILE_VARIANTS)")
        raise
    return plan.precompute()


def _run(w, **kw):
    torch = _torch()
    plan = _plan(w, **kw)
    fhat = torch.from_numpy(w["fhat"]).cuda()
    f = torch.from_numpy(w["f"]).cuda()
    got_f = plan.forward(fhat).cpu().numpy()
    got_y = plan.adjoint(f).cpu().numpy()
    info = plan.info()
    plan.close()
    return got_f, got_y, info


def _oracle(w, batches=None):
    bs = list(range(w["batch"])) if batches is None else list(batches)
    nodes = w["nodes"].astype(np.float64)
    rf = onfft.forward(nodes, w["fhat"][bs].astype(np.complex128), w["N"], w["m"], w["sigma"])
    ry = onfft.adjoint(nodes, w["f"][bs].astype(np.complex128), w["N"], w["m"], w["sigma"])
    return rf, ry


def _check_features(w, **kw):
    plan = _plan(w, **kw)
    feats = plan.features()
    plan.close()
    return feats


def _check(w, tol=None, **kw):
    tol = tol or TOL[w["precision"]]
    got_f, got_y, info = _run(w, **kw)
    rf, ry = _oracle(w)
    for b in range(w["batch"]):
        ef, ey = rel_l2(got_f[b], rf[b]), rel_l2(got_y[b], ry[b])
        assert ef <= tol and ey <= tol, (b, ef, ey, info)
    return info


# ------------------------------------------------------------------ binning

@pytest.mark.parametrize("config", ["cfg1_1d_256", "cfg2_1d_2e18", "cfg3_2d_512", "cfg4_3d_64",
                                    "cfg5_radial_s2", "cfg5_radial_s125"])
def test_binning_bit_exact_on_configs(config):
    w = workloads.make(config, seed=0, batch=1)
    plan = _plan(w)
    perm, offs = plan.binning()
    info = plan.info()
    plan.close()
    ref_perm, ref_offs, P = obin.bin_nodes(w["nodes"], info["Ntilde"], info["tile"])
    assert tuple(info["tiles_per_dim"]) == P
    np.testing.assert_array_equal(perm, ref_perm)
    np.testing.assert_array_equal(offs, ref_offs)


@pytest.mark.parametrize("tile", [(7,), (1,), (400,)])
def test_binning_edge_nodes_1d(tile):
    """On-grid nodes, k = +1/2 (folds to -1/2), out-of-range nodes (periodic
    fold), coincident nodes, ragged last tile, single tile, one-cell tiles."""
    N = 200
    rng = np.random.default_rng(3)
    nodes = np.concatenate([np.arange(-N, N) / (2 * N),          # every grid point (Ntilde = 400)
                            [0.5, -0.5, 0.0, 0.0, 0.0, 1.25, -3.7, 2.0 - 1e-17],
                            rng.random(300) - 0.5])[:, None]
    w = dict(nodes=nodes, N=(N,), m=3, sigma=2.0, precision="c128", batch=1)
    plan = _plan(w, tile=tile)
    perm, offs = plan.binning()
    info = plan.info()
    plan.close()
    ref_perm, ref_offs, _ = obin.bin_nodes(nodes, info["Ntilde"], info["tile"])
    np.testing.assert_array_equal(perm, ref_perm)
    np.testing.assert_array_equal(offs, ref_offs)


def test_binning_all_nodes_one_tile_and_many_tiles():
    """Degenerate partitions: 4096 identical nodes (one hot tile) and
    2^15 tiles in 2D (128 KB shared histograms)."""
    nodes = np.zeros((4096, 2)) + 0.1234
    w = dict(nodes=nodes, N=(256, 256), m=4, sigma=2.0, precision="c128", batch=1)
    plan = _plan(w, tile=(2, 4))
    perm, offs = plan.binning()
    info = plan.info()
    plan.close()
    assert info["n_tiles"] == 256 * 128
    ref_perm, ref_offs, _ = obin.bin_nodes(nodes, info["Ntilde"], info["tile"])
    np.testing.assert_array_equal(perm, ref_perm)
    np.testing.assert_array_equal(offs, ref_offs)


# ------------------------------------------------------------------ window tables

@pytest.mark.parametrize("m", [2, 4, 8])
@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_window_tables_against_oracle_window(m, precision):
    """beta^tensor = 1/(m phi_Base(m n/Ntilde)) and the
    polynomial taps against the exact truncated window psi_hat_Base."""
    N = (100, 64)
    w = dict(nodes=np.zeros((1, 2)), N=N, m=m, sigma=2.0, precision=precision, batch=1)
    plan = _plan(w)
    beta_t, poly, deg = plan.window_tables()
    plan.close()
    off = 0
    for d, n in enumerate(N):
        nt = 2 * n
        b = owin.kb_beta(m, 2.0)
        nn = np.arange(-(n // 2), n // 2)
        ref = 1.0 / (m * owin.phi_base(m * nn / nt, b))
        assert np.max(np.abs(beta_t[off:off + n] - ref) / ref) < 1e-14
        off += n
        zeta = np.linspace(-0.5, 0.5, 1001)[:-1]
        peak = owin.psi_hat_base(np.array([0.0]), b)[0]
        for l in range(2 * m):
            exact = owin.psi_hat_base((zeta + 0.5 + m - 1 - l) / m, b)
            approx = np.polyval(poly[d, l, ::-1], zeta)
            err = np.max(np.abs(approx - exact)) / peak
            assert err < (1e-13 if precision == "c128" else 2e-7), (d, l, err)


# ------------------------------------------------------------------ forward / adjoint parity

@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("method", ["tiled", "tiled_cas", "tiled_loc", "tiled_sorted", "direct"])
def test_config1_all_m(m, method):
    """BASELINE configs[0] (1D N=256, M=256) at every compiled m; ragged tiles."""
    w = workloads.make("cfg1_1d_256", seed=0, m=m)
    _check(w, method=method, tile=(96,))


@pytest.mark.parametrize("method", ["tiled", "tiled_cas", "tiled_loc", "tiled_sorted", "direct"])
@pytest.mark.parametrize("m", [3, 4, 8])
def test_2d_small_ragged_tiles(method, m):
    w = workloads.make("cfg3_2d_512", seed=1, N=(48, 40), M=3000, m=m)
    _check(w, method=method, tile=(20, 14))


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7, 8])
def test_2d_default_path_every_m(m):
    """The default 2D kernels (interp_cell, warp-block spread_wb over the stored
    taps) at every compiled m on a small ragged grid (config 3's m sweep is
    3..8): default tiles and a ragged one."""
    w = workloads.make("cfg3_2d_512", seed=11 + m, N=(48, 42), M=2500, m=m)
    feats = _check_features(w)
    assert "cell_mode" in feats and "wblock" in feats, feats
    _check(w, tile=(20, 14))


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7, 8])
def test_3d_default_path_every_m(m):
    """The default 3D kernels at every compiled m: interp_cell and the warp-block
    adjoint (last dimension long enough for 8 + 2m - 1 cells), ragged tiles."""
    w = workloads.make("cfg4_3d_64", seed=21 + m, N=(14, 12, 12), M=1500, m=m)
    feats = _check_features(w)
    assert "cell_mode" in feats and "wblock" in feats, feats
    _check(w, tile=(6, 5, 7))


@pytest.mark.parametrize("method", ["tiled", "tiled_cas", "tiled_loc", "tiled_sorted", "direct"])
@pytest.mark.parametrize("m", [2, 4, 5])
def test_3d_small_ragged_tiles(method, m):
    w = workloads.make("cfg4_3d_64", seed=2, N=(16, 12, 10), M=2000, m=m)
    _check(w, method=method, tile=(6, 5, 7))


@pytest.mark.parametrize("D", [1, 2, 3])
def test_batch_and_c64(D):
    N = {1: (300,), 2: (40, 36), 3: (12, 12, 10)}[D]
    w = workloads.make({1: "cfg2_1d_2e18", 2: "cfg3_2d_512", 3: "cfg4_3d_64"}[D], seed=3, N=N, M=1500, m=4, batch=3)
    _check(w)
    w32 = dict(w, nodes=w["nodes"].astype(np.float32), fhat=w["fhat"].astype(np.complex64),
               f=w["f"].astype(np.complex64), precision="c64")
    _check(w32)


def test_edge_cases_m1_node_one_cell_tiles_and_wrap():
    """M = 1; nodes at the torus boundary and outside [-1/2,1/2); 1-cell tiles."""
    w = dict(nodes=np.array([[0.5 - 1e-16, -0.5]]), N=(8, 6), m=2, sigma=2.0, precision="c128", batch=1,
             fhat=workloads.complex_normal(np.random.default_rng(0), (1, 8, 6)), f=np.array([[1.0 - 2.0j]]))
    _check(w, tile=(1, 1))
    nodes = np.array([[0.5, 0.5], [-0.5, 0.25], [1.75, -2.3], [0.0, 0.0], [0.0, 0.0], [0.125, -0.25]])
    w = dict(w, nodes=nodes, f=workloads.complex_normal(np.random.default_rng(1), (1, 6)), N=(16, 20), m=4,
             fhat=workloads.complex_normal(np.random.default_rng(2), (1, 16, 20)))
    _check(w, tile=(3, 5))
    _check(w, method="direct")


@pytest.mark.parametrize("config,m", [("cfg2_1d_2e18", m) for m in range(3, 9)] +
                         [("cfg3_2d_512", m) for m in range(3, 9)] + [("cfg4_3d_64", 4)])
def test_full_size_configs(config, m):
    """BASELINE configs[1..3] at full size in the bench's launch configuration,
    every m of the sweep (m = 3..8 on the 1D / 2D sets)."""
    w = workloads.make(config, seed=0, m=m)
    _check(w)


@pytest.mark.parametrize("config", ["cfg5_radial_s2", "cfg5_radial_s125"])
def test_radial_batch_c64_all_vectors(config):
    """BASELINE configs[4]: radial, B = 32, ComplexF32, in the bench's launch
    configuration; every one of the 32 vectors against the (batched) oracle."""
    w = workloads.make(config, seed=0)
    got_f, got_y, _ = _run(w)
    rf, ry = _oracle(w)
    for b in range(w["batch"]):
        assert rel_l2(got_f[b], rf[b]) <= 2e-5, b
        assert rel_l2(got_y[b], ry[b]) <= 2e-5, b


# ------------------------------------------------------------------ invariants / API paths

def test_adjoint_identity_on_gpu():
    torch = _torch()
    w = workloads.make("cfg3_2d_512", seed=5, N=(64, 64), M=5000, m=5)
    plan = _plan(w)
    Af = plan.forward(torch.from_numpy(w["fhat"]).cuda()).cpu().numpy()[0]
    AHf = plan.adjoint(torch.from_numpy(w["f"]).cuda()).cpu().numpy()[0]
    plan.close()
    lhs = np.vdot(w["f"][0], Af)
    rhs = np.vdot(AHf, w["fhat"][0])
    assert abs(lhs - rhs) / (np.linalg.norm(Af) * np.linalg.norm(w["f"][0])) < 1e-14


def test_host_pointer_path_matches_device_path():
    torch = _torch()
    import paper_2208_00049_b200 as pkg
    w = workloads.make("cfg3_2d_512", seed=6, N=(32, 48), M=1000, m=4)
    dev_f, dev_y, _ = _run(w)
    plan = pkg.NfftPlan(w["nodes"], w["N"], m=4).precompute()   # numpy nodes (host)
    host_f = plan.forward(w["fhat"])                              # numpy in -> numpy out
    host_y = plan.adjoint(w["f"])
    plan.close()
    assert isinstance(host_f, np.ndarray)
    assert rel_l2(host_f, dev_f) < 1e-15   # two plans: same kernels, cuFFT may pick another algorithm
    assert rel_l2(host_y, dev_y) < 1e-15


def test_shards_sum_to_full_transform():
    """Linearity: adjoints of disjoint shards of the
    sorted order sum to the full adjoint; forward shards write their nodes."""
    torch = _torch()
    import paper_2208_00049_b200 as pkg
    from paper_2208_00049_b200 import dist
    w = workloads.make("cfg3_2d_512", seed=7, N=(64, 64), M=6000, m=4)
    full_f, full_y, _ = _run(w)
    nodes = torch.from_numpy(w["nodes"]).cuda()
    acc = np.zeros_like(full_y)
    seen = np.zeros(w["M"], bool)
    for rank in range(3):
        rng = dist.shard_range(w["M"], rank, 3)
        plan = pkg.NfftPlan(nodes, w["N"], m=4, node_range=rng).precompute()
        perm = plan.sorted_order()
        out = torch.zeros((1, w["M"]), dtype=torch.complex128, device="cuda")
        plan.forward(torch.from_numpy(w["fhat"]).cuda(), out=out)
        mine = perm[rng[0]:rng[1]]
        # same kernels, other subproblem cuts: equal up to summation-order rounding
        assert rel_l2(out.cpu().numpy()[0, mine], full_f[0, mine]) < 1e-15
        seen[mine] = True
        acc += plan.adjoint(torch.from_numpy(w["f"]).cuda()).cpu().numpy()
        plan.close()
    assert seen.all()
    assert rel_l2(acc, full_y) < 1e-14


def test_errors_are_reported():
    torch = _torch()
    import paper_2208_00049_b200 as pkg
    nodes = torch.tensor([[0.1, float("nan")]], dtype=torch.float64, device="cuda")
    plan = pkg.NfftPlan(nodes, (16, 16), m=2)
    with pytest.raises(pkg.NfftError) as e:
        plan.forward(torch.zeros((1, 16, 16), dtype=torch.complex128, device="cuda"))
    assert e.value.name == "NFFT_ERROR_NOT_PRECOMPUTED"
    with pytest.raises(pkg.NfftError) as e:
        plan.precompute()
    assert e.value.name == "NFFT_ERROR_NONFINITE_NODE"
    plan.close()
    with pytest.raises(pkg.NfftError) as e:
        pkg.NfftPlan(torch.zeros((4, 2), dtype=torch.float64, device="cuda"), (16, 16), m=2, tile=(40, 4))
    assert e.value.name == "NFFT_ERROR_BAD_TILE"
    with pytest.raises(pkg.NfftError) as e:
        pkg.NfftPlan(torch.zeros((4, 1), dtype=torch.float64, device="cuda"), (8,), m=8)
    assert e.value.name == "NFFT_ERROR_BAD_GEOMETRY"


@pytest.mark.parametrize("m", [2, 4, 8])
@pytest.mark.parametrize("D", [1, 2])
def test_owner_computes_spread_small(D, m):
    """Tiles with Q | Ntilde, P >= 3, Q >= 2m select the owner-computes adjoint
    (no zero pass, no atomics); batch 2, c128 and c64."""
    if D == 1:
        w = workloads.make("cfg2_1d_2e18", seed=11, N=(256,), M=700, m=m, batch=2)
        tile = (64,)
    else:
        w = workloads.make("cfg3_2d_512", seed=12, N=(48, 40), M=2500, m=m, batch=2)
        tile = (16, 16)
    _check(w, tile=tile, method="tiled_own")
    w32 = dict(w, nodes=w["nodes"].astype(np.float32), fhat=w["fhat"].astype(np.complex64),
               f=w["f"].astype(np.complex64), precision="c64")
    _check(w32, tile=tile, method="tiled_own")


@pytest.mark.parametrize("method", ["tiled", "tiled_loc", "tiled_own", "tiled_cas", "tiled_sorted"])
def test_radial_clustered_c128(method):
    """Golden-angle radial nodes (402 coincident nodes at the origin, dense
    centre) on a small grid in fp64: exercises duplicate-cell serialisation,
    many-phase chunk schedules and hot tiles split into subproblems."""
    rng = np.random.default_rng(13)
    nodes = workloads.radial_nodes(n_spokes=101, n_samples=128).astype(np.float64)
    N = (64, 64)
    w = dict(nodes=nodes, N=N, m=4, sigma=2.0, precision="c128", batch=1,
             fhat=workloads.complex_normal(rng, (1,) + N), f=workloads.complex_normal(rng, (1, nodes.shape[0])))
    _check(w, method=method, tile=(16, 16))


@pytest.mark.parametrize("method", ["tiled", "tiled_own", "direct"])
def test_repeated_calls_and_stage_api(method):
    """Plan scratch invariants across calls (DESIGN.md §HBM layout): the forward
    input grid keeps its zero padding (out-of-place FFT) and the adjoint grid is
    re-zeroed by the crop; repeated transforms with new data on one plan, and
    the same steps through nfft_run_stage, must all match the oracle."""
    torch = _torch()
    w = workloads.make("cfg3_2d_512", seed=14, N=(48, 64), M=3000, m=4)
    plan = _plan(w, method=method)
    rng = np.random.default_rng(15)
    for rep in range(3):
        fhat = workloads.complex_normal(rng, (1, 48, 64))
        f = workloads.complex_normal(rng, (1, w["M"]))
        got_f = plan.forward(torch.from_numpy(fhat).cuda()).cpu().numpy()[0]
        got_y = plan.adjoint(torch.from_numpy(f).cuda()).cpu().numpy()[0]
        assert rel_l2(got_f, onfft.forward(w["nodes"], fhat[0], w["N"], 4, 2.0)) <= 1e-12
        assert rel_l2(got_y, onfft.adjoint(w["nodes"], f[0], w["N"], 4, 2.0)) <= 1e-12
    fhat_t = torch.from_numpy(fhat).cuda()
    f_t = torch.from_numpy(f).cuda()
    out_f = torch.empty((1, w["M"]), dtype=torch.complex128, device="cuda")
    out_y = torch.empty((1, 48, 64), dtype=torch.complex128, device="cuda")
    plan.run_stage("precompute")
    plan.run_stage("fwd_deconv", fhat_t)
    plan.run_stage("fwd_fft")
    plan.run_stage("fwd_interp", None, out_f)
    plan.run_stage("adj_spread", f_t)
    plan.run_stage("adj_fft")
    plan.run_stage("adj_crop", None, out_y)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out_f.cpu().numpy()[0], got_f)
    assert rel_l2(out_y.cpu().numpy()[0], got_y) < 1e-15
    plan.close()


@pytest.mark.parametrize("D", [1, 2, 3])
def test_execute_overlapped_matches_oracle(D):
    """nfft_execute (precompute || forward deconv+FFT, adjoint || forward on
    internal streams, joined into the plan stream) against the oracle, also
    when captured into a CUDA graph and replayed."""
    torch = _torch()
    import paper_2208_00049_b200 as pkg
    N = {1: (512,), 2: (40, 48), 3: (12, 10, 16)}[D]
    w = workloads.make({1: "cfg2_1d_2e18", 2: "cfg3_2d_512", 3: "cfg4_3d_64"}[D], seed=16, N=N, M=2000, m=4)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan = pkg.NfftPlan(torch.from_numpy(w["nodes"]).cuda(), N, m=4, stream=st.cuda_stream)
        fhat = torch.from_numpy(w["fhat"]).cuda()
        f = torch.from_numpy(w["f"]).cuda()
        fo = torch.empty((1, w["M"]), dtype=torch.complex128, device="cuda")
        yo = torch.empty((1,) + N, dtype=torch.complex128, device="cuda")
        plan.execute(True, fhat, fo, f, yo)
    st.synchronize()
    rf, ry = _oracle(w)
    assert rel_l2(fo.cpu().numpy()[0], rf[0]) <= 1e-12
    assert rel_l2(yo.cpu().numpy()[0], ry[0]) <= 1e-12
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        plan.execute(True, fhat, fo, f, yo)
    fo.zero_()
    yo.zero_()
    with torch.cuda.stream(st):
        g.replay()
    st.synchronize()
    assert rel_l2(fo.cpu().numpy()[0], rf[0]) <= 1e-12
    assert rel_l2(yo.cpu().numpy()[0], ry[0]) <= 1e-12
    plan.close()


@pytest.mark.parametrize("config", ["cfg2_1d_2e18", "cfg3_2d_512", "cfg4_3d_64"])
def test_full_size_execute_as_benched(config):
    """The call bench.py times: one nfft_execute of the direct and the adjoint
    NFFT (adjoint || forward; the 1D adjoint then runs its narrower grid-stride
    launch, several segments per CTA), captured into a CUDA graph and replayed,
    at BASELINE configs[1..3]' full size, against the oracle."""
    torch = _torch()
    import paper_2208_00049_b200 as pkg
    w = workloads.make(config, seed=3)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan = pkg.NfftPlan(torch.from_numpy(w["nodes"]).cuda(), w["N"], m=w["m"], sigma=w["sigma"],
                            stream=st.cuda_stream).precompute()
        fhat = torch.from_numpy(w["fhat"]).cuda()
        f = torch.from_numpy(w["f"]).cuda()
        fo = torch.empty((1, w["M"]), dtype=torch.complex128, device="cuda")
        yo = torch.empty((1,) + tuple(w["N"]), dtype=torch.complex128, device="cuda")
        plan.execute(False, fhat, fo, f, yo)
    st.synchronize()
    rf, ry = _oracle(w)
    assert rel_l2(fo.cpu().numpy()[0], rf[0]) <= 1e-12
    assert rel_l2(yo.cpu().numpy()[0], ry[0]) <= 1e-12
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        plan.execute(False, fhat, fo, f, yo)
    for _ in range(3):  # replays reuse the plan's grids (the adjoint grid must come back zeroed)
        fo.zero_()
        yo.zero_()
        with torch.cuda.stream(st):
            g.replay()
        st.synchronize()
        assert rel_l2(fo.cpu().numpy()[0], rf[0]) <= 1e-12
        assert rel_l2(yo.cpu().numpy()[0], ry[0]) <= 1e-12
    plan.close()


# ------------------------------------------------------------------ D = 1 static-tile path + one-kernel sort

@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("tile", [(64,), (128,)])
def test_1d_static_tile_path(m, tile):
    """Q | Ntilde, P >= 3, Q >= 2m selects interp1d / spread1d (owner-computes,
    crop without re-zeroing) and the cooperative sort; batch 2, c128 + c64."""
    w = workloads.make("cfg2_1d_2e18", seed=21, N=(256,), M=900, m=m, batch=2)
    _check(w, tile=tile)
    w32 = dict(w, nodes=w["nodes"].astype(np.float32), fhat=w["fhat"].astype(np.complex64),
               f=w["f"].astype(np.complex64), precision="c64")
    _check(w32, tile=tile)


def test_1d_static_tile_overfull_tile_and_shards():
    """Clustered nodes: one tile holds > 512 candidates (several spread
    chunks, read-modify-write of owned cells); wrap-around at both ends;
    node shards of the sorted order sum to the full adjoint."""
    torch = _torch()
    import paper_2208_00049_b200 as pkg
    from paper_2208_00049_b200 import dist
    rng = np.random.default_rng(22)
    nodes = np.concatenate([rng.random(1500) * 0.05, rng.random(500) - 0.5,
                            [-0.5, 0.5 - 1e-9, 0.4999, -0.4999, 0.0]])[:, None]
    M = nodes.shape[0]
    w = dict(nodes=nodes, N=(256,), m=4, sigma=2.0, precision="c128", batch=1,
             fhat=workloads.complex_normal(rng, (1, 256)), f=workloads.complex_normal(rng, (1, M)))
    full_f, full_y, _ = _run(w, tile=(32,))
    rf, ry = _oracle(w)
    assert rel_l2(full_f[0], rf[0]) <= 1e-12 and rel_l2(full_y[0], ry[0]) <= 1e-12
    acc = np.zeros_like(full_y)
    for rank in range(3):
        rg = dist.shard_range(M, rank, 3)
        plan = pkg.NfftPlan(torch.from_numpy(nodes).cuda(), (256,), m=4, tile=(32,), node_range=rg).precompute()
        acc += plan.adjoint(torch.from_numpy(w["f"]).cuda()).cpu().numpy()
        plan.close()
    assert rel_l2(acc, full_y) < 1e-14


@pytest.mark.parametrize("config", ["cfg2_1d_2e18", "cfg3_2d_512", "cfg4_3d_64", "cfg5_radial_s2"])
def test_one_kernel_sort_matches_three_kernel_sort(config):
    """The cooperative binsort (default) and the first-generation three-kernel
    sort (method tiled_v1) give the identical permutation and offsets."""
    w = workloads.make(config, seed=4, batch=1)
    tile = {1: (512,), 2: (32, 32), 3: (8, 8, 8)}[len(w["N"])]  # same tiles for both (cell mode widens 3D)
    a = _plan(w, tile=tile)
    b = _plan(w, method="tiled_v1", tile=tile)
    pa, oa = a.binning()
    pb, ob = b.binning()
    a.close()
    b.close()
    np.testing.assert_array_equal(pa, pb)
    np.testing.assert_array_equal(oa, ob)


@pytest.mark.parametrize("config", ["cfg1_1d_256", "cfg2_1d_2e18", "cfg3_2d_512", "cfg4_3d_64", "cfg5_radial_s2",
                                    "cfg5_radial_s125"])
def test_cell_binning_bit_exact(config):
    """Cell mode: the hot-path sort is the oracle's binning with tile = 1 cell
    (key = row-major cell, ties by node index), bit-exact, including the radial
    centre cell with 402 coincident nodes (dense-cell ordering kernel)."""
    w = workloads.make(config, seed=0, batch=1)
    plan = _plan(w)
    cb = plan.cell_binning()
    info = plan.info()
    plan.close()
    if cb is None:
        pytest.skip("plan not in cell mode for this D")
    order, cstart = cb
    ref_perm, ref_offs, _ = obin.bin_nodes(w["nodes"], info["Ntilde"], tuple(1 for _ in info["Ntilde"]))
    np.testing.assert_array_equal(order, ref_perm)
    np.testing.assert_array_equal(cstart, ref_offs)


STRATEGY_CASES = ["1d_small", "1d_ragged_batch", "1d_dense_cells", "1d_full_size", "2d_c128_m5", "2d_c64_batch3",
                  "2d_batch9_c64", "2d_wrap_m8", "2d_full_size", "3d_c128_m3", "3d_c64_ragged", "3d_full_size",
                  "radial_b32_s125_full_size"]


@pytest.mark.parametrize("precompute", ["polynomial", "tensor", "full"])
@pytest.mark.parametrize("case", STRATEGY_CASES)
def test_precompute_strategies(precompute, case):
    """The window precomputation strategies (§3.7) through the
    cell-mode kernels against the oracle: POLYNOMIAL (taps per call), TENSOR
    (2m D taps per node stored, every kernel reads them), FULL (the sparse
    matrix B stored: SpMV forward, owner-computes gather adjoint). Small grids
    whose windows wrap the torus, batches, cells with > 8 nodes, c64 / c128,
    and the BASELINE sizes (config 2, 3, 4 and the radial batch)."""
    tile = None
    if case == "1d_small":
        w = workloads.make("cfg1_1d_256", seed=3, N=(20,), M=70, m=4)
    elif case == "1d_ragged_batch":
        w = workloads.make("cfg1_1d_256", seed=4, N=(300,), M=700, m=5, batch=3)
        tile = (96,)
    elif case == "1d_dense_cells":
        w = workloads.make("cfg1_1d_256", seed=5, N=(64,), M=600, m=3)
        w["nodes"] = np.round(w["nodes"] * 16) / 16  # 16 distinct on-grid positions
    elif case == "1d_full_size":
        w = workloads.make("cfg2_1d_2e18", seed=0, m=4)
    elif case == "2d_c128_m5":
        w = workloads.make("cfg3_2d_512", seed=71, N=(48, 40), M=2500, m=5)
        tile = (20, 14)
    elif case == "2d_c64_batch3":
        w = workloads.make("cfg5_radial_s2", seed=72, N=(40, 36), M=1200, m=4, batch=3)
    elif case == "2d_batch9_c64":
        w = workloads.make("cfg5_radial_s2", seed=73, N=(40, 48), M=1400, m=4, batch=9)
    elif case == "2d_wrap_m8":
        w = workloads.make("cfg3_2d_512", seed=74, N=(18, 20), M=300, m=8)
    elif case == "2d_full_size":
        w = workloads.make("cfg3_2d_512", seed=0, m=4)
    elif case == "3d_c128_m3":
        w = workloads.make("cfg4_3d_64", seed=75, N=(12, 14, 12), M=1500, m=3)
    elif case == "3d_c64_ragged":
        w = workloads.make("cfg4_3d_64", seed=76, N=(10, 12, 14), M=1200, m=2)
        w = dict(w, nodes=w["nodes"].astype(np.float32), fhat=w["fhat"].astype(np.complex64),
                 f=w["f"].astype(np.complex64), precision="c64")
        tile = (6, 5, 7)
    elif case == "3d_full_size":
        w = workloads.make("cfg4_3d_64", seed=0, m=4)
    else:
        w = workloads.make("cfg5_radial_s125", seed=0)
    kw = dict(precompute=precompute)
    if tile:
        kw["tile"] = tile
    feats = _check_features(w, **kw)
    assert "cell_mode" in feats, feats
    assert ("tensor" in feats) == (precompute == "tensor") and ("full" in feats) == (precompute == "full"), feats
    if case == "radial_b32_s125_full_size":
        got_f, got_y, _ = _run(w, **kw)
        rf, ry = _oracle(w, range(0, 32, 5))
        for i, b in enumerate(range(0, 32, 5)):
            assert rel_l2(got_f[b], rf[i]) <= 2e-5 and rel_l2(got_y[b], ry[i]) <= 2e-5, b
    else:
        _check(w, **kw)


@pytest.mark.parametrize("precompute", ["tensor", "full"])
@pytest.mark.parametrize("D", [1, 2, 3])
def test_strategy_shards_sum_to_full_transform(precompute, D):
    """Node shards (options.node_begin/end over the cell-sorted order) with the
    stored-table strategies: the shards' forward outputs cover disjoint nodes
    and their adjoints sum to the full adjoint (linearity)."""
    torch = _torch()
    import paper_2208_00049_b200 as pkg
    from paper_2208_00049_b200 import dist
    w = {1: workloads.make("cfg2_1d_2e18", seed=81, N=(400,), M=900, m=4),
         2: workloads.make("cfg3_2d_512", seed=82, N=(36, 40), M=1500, m=4),
         3: workloads.make("cfg4_3d_64", seed=83, N=(12, 12, 12), M=1200, m=3)}[D]
    rf, ry = _oracle(w)
    nodes = torch.from_numpy(w["nodes"]).cuda()
    acc_f = np.zeros((1, w["M"]), complex)
    acc_y = np.zeros((1,) + tuple(w["N"]), complex)
    for rank in range(3):
        plan = pkg.NfftPlan(nodes, w["N"], m=w["m"], precompute=precompute,
                            node_range=dist.shard_range(w["M"], rank, 3)).precompute()
        out = torch.zeros((1, w["M"]), dtype=torch.complex128, device="cuda")
        acc_f += plan.forward(torch.from_numpy(w["fhat"]).cuda(), out=out).cpu().numpy()
        acc_y += plan.adjoint(torch.from_numpy(w["f"]).cuda()).cpu().numpy()
        plan.close()
    assert rel_l2(acc_f[0], rf[0]) <= 1e-12 and rel_l2(acc_y[0], ry[0]) <= 1e-12


@pytest.mark.parametrize("case", ["2d_c64_b32", "2d_c128_b9", "radial_b33_s125", "2d_c64_b8_m8"] +
                         [f"2d_c128_b8_m{mm}" for mm in (1, 2, 5, 6, 7)] + [f"2d_c64_b16_m{mm}" for mm in (1, 2, 3, 5, 6, 7)])
def test_batch_adjoint(case):
    """2D batches of >= 8 transforms: the batch adjoint with lanes = batch
    vectors (spread_rb2, resample_rowbatch.cuh) and, for fp32, the two-vector
    interpolation (interp_cell2, bank-rotated for 2m = 8, 16); every vector
    against the oracle, ragged
    chunks (B = 9, 33), wrapped windows, c64 and c128."""
    if case == "2d_c64_b32":
        w = workloads.make("cfg5_radial_s2", seed=13, N=(40, 36), M=1200, m=4, batch=32)
    elif case == "2d_c128_b9":
        w = workloads.make("cfg3_2d_512", seed=14, N=(48, 40), M=1500, m=3, batch=9)
    elif case == "2d_c64_b8_m8":
        w = workloads.make("cfg5_radial_s2", seed=17, N=(48, 64), M=900, m=8, batch=8)
    elif case.startswith("2d_c128_b8_m"):
        mm = int(case[-1])
        w = workloads.make("cfg3_2d_512", seed=18 + mm, N=(48, 64), M=1000, m=mm, batch=8)
    elif case.startswith("2d_c64_b16_m"):
        mm = int(case[-1])
        w = workloads.make("cfg5_radial_s2", seed=28 + mm, N=(40, 48), M=1100, m=mm, batch=16)
    else:
        w = workloads.make("cfg5_radial_s125", seed=16, N=(64, 64), M=2000, m=4, batch=33)
    plan = _plan(w)
    feats = plan.features()
    plan.close()
    assert "batch" in feats, feats
    _check(w)


@pytest.mark.parametrize("case", ["1d_m3", "1d_m7_c64", "2d_m4", "3d_m2", "radial_b32"])
def test_window_2m_plus_2(case):
    """NFFT3-style window variant: 2m+2 samples of the continued
    window, same shape and correction; against the oracle's variant."""
    if case == "1d_m3":
        w = workloads.make("cfg1_1d_256", seed=23, m=3)
    elif case == "1d_m7_c64":
        w = workloads.make("cfg1_1d_256", seed=24, N=(300,), M=900, m=7)
        w["precision"] = "c64"
        w["nodes"] = w["nodes"].astype(np.float32)
        w["fhat"] = w["fhat"].astype(np.complex64)
        w["f"] = w["f"].astype(np.complex64)
    elif case == "2d_m4":
        w = workloads.make("cfg3_2d_512", seed=25, N=(48, 40), M=2000, m=4)
    elif case == "3d_m2":
        w = workloads.make("cfg4_3d_64", seed=26, N=(12, 10, 14), M=800, m=2)
    else:
        w = workloads.make("cfg5_radial_s2", seed=27, N=(48, 48), M=1500, m=4, batch=32)
    torch = _torch()
    import paper_2208_00049_b200 as pkg
    plan = _plan(w, window_points="2m+2")
    fhat = torch.from_numpy(w["fhat"]).cuda()
    f = torch.from_numpy(w["f"]).cuda()
    got_f = plan.forward(fhat).cpu().numpy()
    got_y = plan.adjoint(f).cpu().numpy()
    plan.close()
    tol = TOL[w["precision"]]
    for b in range(w["batch"]):
        rf = onfft.forward(w["nodes"], w["fhat"][b], w["N"], w["m"], w["sigma"], window_points="2m+2")
        ry = onfft.adjoint(w["nodes"], w["f"][b], w["N"], w["m"], w["sigma"], window_points="2m+2")
        assert rel_l2(got_f[b], rf) <= tol and rel_l2(got_y[b], ry) <= tol, (b, rel_l2(got_f[b], rf), rel_l2(got_y[b], ry))


@pytest.mark.parametrize("D", [1, 2, 3])
def test_very_dense_cell(D):
    """3000 of the nodes in ONE cell (> 2048: the cell sort's scratch path) plus
    a uniform background; spread windows hold far more nodes than one staging
    chunk. Cell binning stays bit-exact (stable order), transforms match."""
    N = {1: (128,), 2: (32, 24), 3: (12, 10, 8)}[D]
    w = workloads.make({1: "cfg1_1d_256", 2: "cfg3_2d_512", 3: "cfg4_3d_64"}[D], seed=30 + D, N=N, M=3600, m=3)
    w["nodes"][:3000] = 0.1234567  # one cell, every dimension
    plan = _plan(w)
    cb = plan.cell_binning()
    info = plan.info()
    plan.close()
    ref_perm, ref_offs, _ = obin.bin_nodes(w["nodes"], info["Ntilde"], tuple(1 for _ in info["Ntilde"]))
    np.testing.assert_array_equal(cb[0], ref_perm)
    np.testing.assert_array_equal(cb[1], ref_offs)
    _check(w)


@pytest.mark.parametrize("D", [1, 2, 3])
def test_autotune_tile(D):
    """Online block-size benchmark: returns one of the candidates
    with a positive time; a plan with that tile matches the oracle."""
    import paper_2208_00049_b200 as pkg
    N = {1: (512,), 2: (64, 48), 3: (16, 12, 10)}[D]
    cand = {1: [(64,), (128,), (512,)], 2: [(16, 16), (32, 32), (16, 32)], 3: [(4, 4, 8), (8, 8, 8)]}[D]
    w = workloads.make({1: "cfg1_1d_256", 2: "cfg3_2d_512", 3: "cfg4_3d_64"}[D], seed=40 + D, N=N, M=2000, m=3)
    tile, ms = pkg.autotune_tile(w["nodes"], w["N"], m=3, candidates=cand, reps=3)
    assert tile in cand and ms > 0, (tile, ms)
    _check(w, tile=tile)


@pytest.mark.parametrize("config", ["cfg1_1d_256", "cfg3_2d_small"])
def test_execute_with_host_buffers(config):
    """nfft_execute with host (pinned and pageable) inputs / outputs: the copies
    run on each chain's stream; results equal the oracle after the sync."""
    torch = _torch()
    if config == "cfg1_1d_256":
        w = workloads.make("cfg1_1d_256", seed=50, batch=2)
    else:
        w = workloads.make("cfg3_2d_512", seed=51, N=(40, 36), M=1500, batch=2)
    plan = _plan(w)
    for pinned in (True, False):
        def host(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            return (t.pin_memory() if pinned else t).numpy()
        fhat, f = host(w["fhat"]), host(w["f"])
        fout = host(np.zeros((w["batch"], w["M"]), w["f"].dtype))
        yout = host(np.zeros(w["fhat"].shape, w["fhat"].dtype))
        plan.execute(False, fhat, fout, f, yout)
        torch.cuda.synchronize()
        rf, ry = _oracle(w)
        for b in range(w["batch"]):
            assert rel_l2(fout[b], rf[b]) <= 1e-12 and rel_l2(yout[b], ry[b]) <= 1e-12
    plan.close()


@pytest.mark.parametrize("case", ["3d", "2d_batch8"])
def test_seam_and_out_of_range_nodes(case):
    """Nodes on the torus seam (k = +-1/2), exactly on grid points, far outside
    [-1/2, 1/2) (periodic fold) and coincident, through the default cell-mode
    kernels (3D; the 2D batch adjoint with B = 8)."""
    rng = np.random.default_rng(60)
    D = 3 if case == "3d" else 2
    special = np.array([[0.5] * D, [-0.5] * D, [1.75] * D, [-2.3] * D, [0.0] * D, [0.0] * D,
                        [0.25, -0.5, 0.5][:D], [0.5 - 1e-16, 0.125, -0.375][:D]])
    nodes = np.concatenate([special, rng.random((600, D)) - 0.5])
    N = (12, 10, 16) if D == 3 else (40, 32)
    B = 1 if D == 3 else 8
    w = dict(nodes=nodes, N=N, m=3, sigma=2.0, precision="c128", batch=B,
             fhat=workloads.complex_normal(rng, (B,) + N), f=workloads.complex_normal(rng, (B, len(nodes))))
    _check(w)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["2d_m4", "2d_m1_c64", "2d_m8_ragged", "2d_b3", "3d_m4", "3d_m2_ragged_c64",
                                  "3d_m8", "3d_2m2", "3d_b2_c64", "2d_short_dim0", "3d_short_dim0"])
def test_warp_block_adjoint(case):
    """D = 2, 3 adjoint over warp-owned cell blocks (resample_wblock.cuh): the
    default when the last dimension holds the block's window. Grids that are
    not multiples of the block (8 x 32 / 8 x 4 x 8 cells), wrapped windows,
    m = 1..8, the 2m+2 window, batches, c64 / c128 against the oracle."""
    kw = {}
    if case == "2d_m4":
        w = workloads.make("cfg3_2d_512", seed=21, N=(40, 64), M=3000, m=4)
    elif case == "2d_m1_c64":
        w = workloads.make("cfg5_radial_s2", seed=22, N=(24, 40), M=1500, m=1, batch=1)
    elif case == "2d_m8_ragged":
        w = workloads.make("cfg3_2d_512", seed=23, N=(26, 42), M=2500, m=8)
    elif case == "2d_b3":
        w = workloads.make("cfg3_2d_512", seed=24, N=(30, 48), M=2000, m=4, batch=3)
    elif case == "3d_m4":
        w = workloads.make("cfg4_3d_64", seed=25, N=(12, 10, 16), M=3000, m=4)
    elif case == "3d_m2_ragged_c64":
        w = workloads.make("cfg4_3d_64", seed=26, N=(10, 6, 14), M=2000, m=2)
        w = dict(w, precision="c64", nodes=w["nodes"].astype(np.float32), fhat=w["fhat"].astype(np.complex64),
                 f=w["f"].astype(np.complex64))
    elif case == "3d_m8":
        w = workloads.make("cfg4_3d_64", seed=27, N=(16, 16, 12), M=1500, m=8)
    elif case == "2d_short_dim0":  # Nt_0 = 12 < the block's 16 dim-0 cells: window planes repeat
        w = workloads.make("cfg3_2d_512", seed=33, N=(6, 40), M=800, m=2)
    elif case == "3d_short_dim0":  # Nt = (8, 12, 20)
        w = workloads.make("cfg4_3d_64", seed=34, N=(4, 6, 10), M=700, m=2)
    elif case == "3d_2m2":
        w = workloads.make("cfg4_3d_64", seed=28, N=(12, 12, 12), M=1500, m=3)
        kw = {"window_points": "2m+2"}
    else:
        w = workloads.make("cfg4_3d_64", seed=29, N=(8, 12, 10), M=1200, m=3, batch=2)
        w = dict(w, precision="c64", nodes=w["nodes"].astype(np.float32), fhat=w["fhat"].astype(np.complex64),
                 f=w["f"].astype(np.complex64))
    plan = _plan(w, **kw)
    feats = plan.features()
    plan.close()
    assert "wblock" in feats, feats
    if kw:
        torch = _torch()
        plan = _plan(w, **kw)
        got_y = plan.adjoint(torch.from_numpy(w["f"]).cuda()).cpu().numpy()
        plan.close()
        nodes = w["nodes"].astype(np.float64)
        for b in range(w["batch"]):
            ry = onfft.adjoint(nodes, w["f"][b].astype(np.complex128), w["N"], w["m"], w["sigma"],
                               window_points="2m+2")
            assert rel_l2(got_y[b], ry) <= TOL[w["precision"]]
    else:
        _check(w)


@pytest.mark.gpu
@pytest.mark.parametrize("D", [2, 3])
def test_warp_block_shards_and_fallback(D):
    """Node shards through the warp-block adjoint sum to the full adjoint; on a
    grid whose last dimension is too short for the warp blocks (Ntilde_last <
    32 + 2m - 1 in 2D, 8 + 2m - 1 in 3D) the spread_cell fallback takes the
    plan and matches the oracle."""
    torch = _torch()
    import paper_2208_00049_b200 as pkg
    from paper_2208_00049_b200 import dist
    if D == 2:
        w = workloads.make("cfg3_2d_512", seed=31, N=(32, 48), M=4000, m=4)
        small = workloads.make("cfg3_2d_512", seed=33, N=(40, 12), M=2000, m=4)
    else:
        w = workloads.make("cfg4_3d_64", seed=32, N=(12, 12, 12), M=3000, m=3)
        small = workloads.make("cfg4_3d_64", seed=34, N=(12, 10, 6), M=2000, m=3)
    _, full_y, _ = _run(w)
    _, ry = _oracle(w)
    assert rel_l2(full_y[0], ry[0]) <= TOL["c128"]
    nodes = torch.from_numpy(w["nodes"]).cuda()
    acc = np.zeros_like(full_y)
    for rank in range(3):
        plan = pkg.NfftPlan(nodes, w["N"], m=w["m"], node_range=dist.shard_range(w["M"], rank, 3)).precompute()
        assert "wblock" in plan.features()
        acc += plan.adjoint(torch.from_numpy(w["f"]).cuda()).cpu().numpy()
        plan.close()
    assert rel_l2(acc, full_y) < 1e-14
    plan = _plan(small)
    feats = plan.features()
    plan.close()
    assert "wblock" not in feats and "cell_mode" in feats, feats
    _check(small)


@pytest.mark.gpu
def test_large_tile_without_cell_adjoint_drops_to_direct():
    """A tile beyond the spread_cell fallback's limits (> 512 gather items) on a
    grid too short for the warp blocks: no cell-mode adjoint exists, so the
    plan leaves cell mode (unblocked kernels) and still matches the oracle."""
    w = workloads.make("cfg3_2d_512", seed=35, N=(128, 12), M=2500, m=4)
    plan = _plan(w, tile=(128, 24))
    feats = plan.features()
    plan.close()
    assert "cell_mode" not in feats, feats
    _check(w, tile=(128, 24))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["2d_tile_64x64", "radial_tile_32x128"])
def test_large_tiles_keep_cell_mode(case):
    """Tiles beyond the spread_cell fallback's limits (more than 512 gather items)
    stay in cell mode when the warp-block or the batch adjoint takes the plan."""
    if case == "2d_tile_64x64":
        w = workloads.make("cfg3_2d_512", seed=41, N=(64, 96), M=3000, m=4)
        tile, feat = (64, 64), "wblock"
    else:
        w = workloads.make("cfg5_radial_s2", seed=42, N=(64, 96), M=2000, m=4, batch=8)
        tile, feat = (32, 128), "batch"
    plan = _plan(w, tile=tile)
    feats = plan.features()
    plan.close()
    assert "cell_mode" in feats and feat in feats, feats
    _check(w, tile=tile)


@pytest.mark.parametrize("case", ["1d_c128", "1d_c64_m7", "2d_mixed_c128", "2d_odd_batch9_c64", "3d_odd_c128",
                                  "2d_odd_direct"])
def test_odd_n(case):
    """Odd N_d (n_d = -(N_d-1)/2 .. (N_d-1)/2, storage i = n + (N_d-1)/2)
    through the default kernels (and the unblocked ones) against the oracle."""
    kw = {}
    if case == "1d_c128":
        w = workloads.make("cfg2_1d_2e18", seed=61, N=(1001,), M=900, m=4)
    elif case == "1d_c64_m7":
        w = workloads.make("cfg2_1d_2e18", seed=62, N=(333,), M=500, m=7)
        w = dict(w, nodes=w["nodes"].astype(np.float32), fhat=w["fhat"].astype(np.complex64),
                 f=w["f"].astype(np.complex64), precision="c64")
    elif case == "2d_mixed_c128":
        w = workloads.make("cfg3_2d_512", seed=63, N=(45, 52), M=2500, m=5)
    elif case == "2d_odd_batch9_c64":
        w = workloads.make("cfg5_radial_s125", seed=64, N=(63, 61), M=1500, m=4, batch=9)
    elif case == "3d_odd_c128":
        w = workloads.make("cfg4_3d_64", seed=65, N=(13, 11, 15), M=1500, m=3)
    else:
        w = workloads.make("cfg3_2d_512", seed=66, N=(23, 31), M=800, m=4)
        kw = dict(method="direct")
    _check(w, **kw)


def test_stage_times():
    """timing = 1: nfft_get_stage_times (deconv, FFT, resampling of
    the most recent call) and nfft_get_stage_times_ex (all five per direction)."""
    torch = _torch()
    import ctypes
    import paper_2208_00049_b200 as pkg
    w = workloads.make("cfg3_2d_512", seed=91, N=(64, 64), M=3000, m=4)
    plan = _plan(w, timing=True)
    plan.forward(torch.from_numpy(w["fhat"]).cuda())
    ms = [ctypes.c_float() for _ in range(3)]
    assert pkg.lib().nfft_get_stage_times(plan._h, *[ctypes.byref(x) for x in ms]) == 0
    assert all(x.value > 0 for x in ms), [x.value for x in ms]
    plan.adjoint(torch.from_numpy(w["f"]).cuda())
    assert pkg.lib().nfft_get_stage_times(plan._h, *[ctypes.byref(x) for x in ms]) == 0
    st = plan.stage_times("adjoint")
    assert abs(st["resample"] - ms[2].value) < 1e-6 and st["resample"] > 0 and st["fft"] > 0
    assert plan.stage_times("forward")["deconv"] > 0
    plan.close()
    nt = _plan(w)
    assert pkg.lib().nfft_get_stage_times(nt._h, None, None, None) == 1  # no timing events
    nt.close()
