"""GPU parity: the sm_100a path (through liblpbp.so's C ABI) against the
reference's golden vectors and the CPU oracle.  Bar: relative L2 <= 1e-4 in
fp32 (BASELINE.json north_star), max-abs reported."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fastbp_oracle as O
from oracle import phantoms

pytestmark = pytest.mark.gpu

RTOL = 1e-4  # north_star: relative L2 <= 1e-4 in fp32


@pytest.fixture(scope="module")
def pkg():
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    import paper_1608_03589_b200 as p
    return p


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def report(name, got, ref):
    r = O.relative_l2(got, ref)
    m = O.max_abs(got, ref)
    print(f"{name}: rel_l2={r:.3e} max_abs={m:.3e}")
    return r


def test_native_library_is_loaded(pkg):
    import ctypes
    from paper_1608_03589_b200 import _native
    lib = _native.lib()
    assert lib._name.endswith("liblpbp.so")


def test_cfg0_backprojection_vs_reference_golden(pkg, golden):
    z = golden("cfg0.npz")
    g = pkg.Sinogram(256, 256, z["sino"].astype(np.float64))
    img = pkg.logpolar_backproject(g, 256)
    assert report("cfg0 bp", img.values, z["bp"]) <= RTOL


def test_cfg0_stages(pkg, golden):
    z = golden("cfg0.npz")
    plan = pkg.get_plan(256, 256, 256, None, None, None)
    lp = plan.logpolar(dev(z["sino"])[None])[0].cpu().numpy()
    assert report("cfg0 logpolar stage", lp, z["lp"]) <= RTOL
    # readout alone, fed the oracle's log-polar image
    ref_lp = O.logpolar_stage(z["sino"].astype(np.float64), 256)
    img = plan.readout(dev(ref_lp)[None])[0].cpu().numpy()
    assert report("cfg0 readout", img, O.lp_readout(ref_lp, plan.rho0, 256, 256)) <= 1e-6


def test_cfg0_fbp_and_filter(pkg, golden):
    z = golden("cfg0.npz")
    g = pkg.Sinogram(256, 256, z["sino"].astype(np.float64))
    f = pkg.filter_sinogram(g, pkg.FilterSpec())
    assert report("cfg0 filter", f.values, z["filtered"]) <= 1e-5
    img = pkg.fbp(g, pkg.FilterSpec(), engine="logpolar", n=256)
    assert report("cfg0 fbp", img.values, z["fbp"]) <= RTOL


def test_cfg1_fbp_batch_vs_oracle(pkg, golden):
    z = golden("cfg1.npz")
    sinos = np.stack([phantoms.config_sinogram(1, i) for i in range(16)])
    assert np.array_equal(sinos[0], z["sino"])
    out = pkg.fbp_batch(dev(sinos), pkg.FilterSpec(), 512).cpu().numpy()
    assert report("cfg1 fbp slice0 vs reference", out[0], z["fbp"]) <= RTOL
    for i in (1, 7, 15):
        ref = O.fbp_logpolar(sinos[i].astype(np.float64), 512)
        assert report(f"cfg1 fbp slice{i} vs oracle", out[i], ref) <= RTOL


def test_tikhonov_cutoff(pkg, golden):
    z = golden("cfg1.npz")
    g = pkg.Sinogram(512, 512, z["sino"].astype(np.float64))
    img = pkg.fbp(g, pkg.FilterSpec(lam=0.02, cutoff=0.9), engine="logpolar", n=512)
    assert report("cfg1 tikhonov", img.values, z["fbp_tik"]) <= RTOL


def test_options_nonsquare_odd(pkg, golden):
    z = golden("opts.npz")
    g = pkg.Sinogram(512, 256, z["sino"].astype(np.float64))
    assert report("opts default", pkg.logpolar_backproject(g, 256).values, z["bp_default"]) <= RTOL
    o = pkg.LogPolarOptions(rho0=-4.0, nrho=600)
    assert report("opts rho0/nrho", pkg.logpolar_backproject(g, 256, o).values, z["bp_opts"]) <= RTOL
    assert report("opts n=300", pkg.logpolar_backproject(g, 300).values, z["bp_n300"]) <= RTOL
    ref = O.logpolar_backproject(z["sino"].astype(np.float64), 255)
    assert report("opts n=255 (odd)", pkg.logpolar_backproject(g, 255).values, ref) <= RTOL


def test_zero_linearity_and_batch_invariance(pkg):
    plan = pkg.get_plan(512, 512, 512, None, None, (0.0, 1.0))
    zero = torch.zeros((2, 512, 512), device="cuda")
    assert torch.count_nonzero(plan.execute(zero)) == 0
    a = dev(phantoms.config_sinogram(1, 3))[None]
    b = dev(phantoms.config_sinogram(1, 4))[None]
    ia, ib = plan.execute(a), plan.execute(b)
    iab = plan.execute(2.0 * a - 0.5 * b)
    assert O.relative_l2((iab).cpu().numpy(), (2.0 * ia - 0.5 * ib).cpu().numpy()) < 1e-5
    # a slice's result does not depend on its batch neighbours or the chunking
    batch = torch.cat([b, a, b, a, a], 0)
    full = plan.execute(batch, chunk=5)
    ch = plan.execute(batch, chunk=2)
    assert torch.equal(full, ch)
    assert torch.equal(full[1], ia[0]) and torch.equal(full[0], ib[0])


def test_host_to_host_matches_device(pkg):
    plan = pkg.get_plan(512, 512, 512, None, None, (0.0, 1.0))
    sinos = np.stack([phantoms.config_sinogram(1, i) for i in range(6)])
    ref = plan.execute(dev(sinos)).cpu().numpy()
    host = torch.from_numpy(sinos).pin_memory()
    out = plan.execute_host(host, chunk=4)
    assert np.array_equal(out.numpy(), ref)
    out2 = plan.execute_host(sinos, chunk=1)
    assert np.array_equal(out2, ref)


@pytest.mark.slow
def test_host_paths_2048_bitwise(pkg):
    """Config-3 geometry (2048^2 FBP): the pipelined host->host path (pinned tensors and numpy,
    ragged chunking) and a VolumeReconstructor with two plans sharding the slices are bitwise
    equal to the device-resident path."""
    ids = [0, 1, 2, 5, 9, 11]
    sinos = torch.stack([torch.from_numpy(phantoms.config_sinogram(3, i)) for i in ids])
    plan = pkg.get_plan(2048, 2048, 2048, None, None, (0.0, 1.0))
    ref = plan.execute(sinos.cuda(), chunk=4).cpu()
    host = sinos.pin_memory()
    assert torch.equal(plan.execute_host(host, chunk=4), ref)
    assert np.array_equal(plan.execute_host(sinos.numpy(), chunk=3), ref.numpy())
    vr = pkg.VolumeReconstructor(2048, 2048, 2048, filter_spec=(0.0, 1.0), devices=[0, 0], chunk=2)
    assert torch.equal(vr.run(host), ref)
    assert np.array_equal(vr.run(sinos.numpy()), ref.numpy())
    with pytest.raises(ValueError):
        plan.execute_host(host, out=torch.empty((6, 2048, 2047)))
    with pytest.raises(ValueError):
        plan.execute(sinos.cuda(), out=torch.empty((6, 2048, 2048), device="cuda", dtype=torch.float64))


@pytest.mark.slow
def test_bench_generated_input_parity(pkg):
    """The benched workload is the parity-tested one: a config-3 slice made by the bench's
    device generator (synth.config_batch), downloaded, reconstructed by the oracle, and compared
    with the GPU FBP of the same device-resident slice."""
    k = 1234
    x = pkg.synth.config_batch(3, [k], torch.device("cuda"))
    g = x[0].cpu().numpy().astype(np.float64)
    out = pkg.fbp_batch(x, pkg.FilterSpec(), 2048)[0].cpu().numpy()
    assert report("bench input slice 1234 fbp", out, O.fbp_logpolar(g, 2048)) <= RTOL
    # and the device generator's noiseless part is the reference's radon_ellipses
    c = pkg.synth.CONFIGS[3]
    prm = pkg.synth.ellipse_params(pkg.synth.BASE_SEED + 7919 * 3 + k, c["k"], c["amin"], c["amax"])
    clean = pkg.synth.radon_ellipses_batch(prm[None], 2048, 2048, torch.device("cuda"),
                                           dtype=torch.float64)[0].cpu().numpy()
    e = phantoms.random_ellipses(pkg.synth.BASE_SEED + 7919 * 3 + k, c["k"], c["amin"], c["amax"])
    assert np.allclose(prm, np.stack([e.cx, e.cy, e.a, e.b, e.tilt, e.rho], axis=1), rtol=0, atol=0)
    assert report("bench input noiseless part", clean, phantoms.radon_ellipses(e, 2048, 2048)) <= 1e-12


def test_naive_backprojector(pkg, golden):
    z = golden("cfg0.npz")
    g = pkg.Sinogram(256, 256, z["sino"].astype(np.float64))
    img = pkg.backproject_naive(g, 256)
    assert report("cfg0 naive", img.values, z["naive"]) <= RTOL
    img = pkg.fbp(g, pkg.FilterSpec(), engine="naive", n=200)
    ref = O.FBP_SCALE * O.backproject_naive(O.ramp_filter(z["sino"].astype(np.float64)), 200)
    assert report("cfg0 fbp naive", img.values, ref) <= RTOL


@pytest.mark.slow
def test_cfg2_full_size_samples(pkg):
    """2048 bins x 2048 angles -> 2048^2 backprojection on sampled slices (oracle ~5 s each)."""
    sinos = np.stack([phantoms.config_sinogram(2, i) for i in (0, 1)])
    out = pkg.logpolar_backproject_batch(dev(sinos), 2048).cpu().numpy()
    for i in range(2):
        ref = O.logpolar_backproject(sinos[i].astype(np.float64), 2048)
        assert report(f"cfg2 slice{i}", out[i], ref) <= RTOL


@pytest.mark.slow
def test_cfg3_fbp_full_size_sample(pkg):
    s = phantoms.config_sinogram(3, 5)
    out = pkg.fbp_batch(dev(s)[None], pkg.FilterSpec(), 2048).cpu().numpy()[0]
    ref = O.fbp_logpolar(s.astype(np.float64), 2048)
    assert report("cfg3 slice5 fbp", out, ref) <= RTOL


def test_unsupported_size_is_loud(pkg):
    g = pkg.Sinogram(64, 5000, np.ones((64, 5000)))  # Bluestein row DFT would need 32768 points
    with pytest.raises(NotImplementedError):
        pkg.logpolar_backproject(g, 64)
    with pytest.raises(NotImplementedError):  # BST: odd nt
        pkg.fbp(pkg.Sinogram(129, 90, np.ones((129, 90))), pkg.FilterSpec(), engine="bst", n=64)


@pytest.mark.slow
@pytest.mark.parametrize("nt,nth", [(3200, 2048), (2048, 3200)])
def test_paper_lnls_sizes(pkg, nt, nth):
    """The paper's motivating workload (reconstructions from 3200 x 2048
    datasets), both orientations, FBP to 2048^2 against the oracle.
    3200 bins x 2048 angles: ns = 1600, nrho = 6096 -> a 16384-point rho FFT and an
    8192-point ramp embedding; 2048 bins x 3200 angles: nphi = 6400 = 25 x 256 -> mixed-radix
    row DFTs (25-point DFTs in registers + 256-point FFTs)."""
    g = phantoms.sinogram(4242 + nt, nt, nth, 50, 0.01, 0.3, 0.01)
    plan = pkg.get_plan(nt, nth, 2048, None, None, (0.0, 1.0))
    assert (plan.info["L"], plan.info["M"]) == ((16384, 8192) if nt == 3200 else (8192, 4096))
    if nth == 3200:  # nphi = 6400 = 25 x 256: mixed-radix row DFTs (Bluestein would run 16384-point convolutions)
        assert plan.info["generic"] == 1 and plan.info["MB"] == 16384 and plan.info["phi_q"] == 25
    out = pkg.fbp_batch(dev(g)[None], pkg.FilterSpec(), 2048)[0].cpu().numpy()
    ref = O.fbp_logpolar(g.astype(np.float64), 2048)
    assert report(f"paper size {nt}x{nth} fbp -> 2048", out, ref) <= RTOL
    bp = pkg.logpolar_backproject_batch(dev(g)[None], 2048)[0].cpu().numpy()
    assert report(f"paper size {nt}x{nth} bp -> 2048", bp, O.logpolar_backproject(g.astype(np.float64), 2048)) <= RTOL


@pytest.mark.parametrize("nt,nth,n,filt", [(129, 90, 64, False), (255, 128, 128, True), (301, 200, 150, False)])
def test_odd_nt(pkg, nt, nth, n, filt):
    """Odd detector counts (the reference accepts any nt >= 2): generic row DFTs, spectra
    columns padded to an even pitch."""
    g = phantoms.sinogram(1100 + nt, nt, nth, 8, 0.05, 0.35, 0.01).astype(np.float64)
    s = pkg.Sinogram(nt, nth, g)
    if filt:
        got = pkg.fbp(s, pkg.FilterSpec(), engine="logpolar", n=n).values
        ref = O.fbp_logpolar(g, n)
    else:
        got = pkg.logpolar_backproject(s, n).values
        ref = O.logpolar_backproject(g, n)
    assert report(f"odd nt {nt}x{nth}->{n} {'fbp' if filt else 'bp'}", got, ref) <= RTOL


def test_device_sinogram_generator_matches_oracle(pkg):
    """synth (device, fp64 line integrals) vs oracle/phantoms (numpy) on noiseless inputs."""
    from paper_1608_03589_b200 import synth
    for cfg, idx in ((0, 0), (2, 3)):
        c = phantoms.CONFIGS[cfg]
        seed = phantoms.BASE_SEED + 7919 * cfg + idx
        prm = synth.ellipse_params(seed, c["k"], c["amin"], c["amax"])
        ref = phantoms.radon_ellipses(phantoms.random_ellipses(seed, c["k"], c["amin"], c["amax"]), c["nt"], c["ntheta"])
        got = synth.radon_ellipses_batch(prm[None], c["nt"], c["ntheta"], torch.device("cuda"))[0].cpu().numpy()
        assert report(f"synth cfg{cfg}", got, ref) < 1e-6


def test_profiled_stage_times_cover_every_stage(pkg):
    plan = pkg.get_plan(512, 512, 512, None, None, (0.0, 1.0))
    x = dev(np.stack([phantoms.config_sinogram(1, i) for i in range(4)]))
    plan.profile(True)
    plan.execute(x, chunk=2)
    st = plan.profile_read()
    plan.profile(False)
    assert set(st) == {"ramp_filter", "row_rdft", "rho_conv", "irdft_readout"}
    assert all(v["launches"] == 2 and v["slices"] == 4 and v["ms"] > 0 for v in st.values())
    assert plan.last_launches == 8


@pytest.mark.parametrize("fbp", [False, True])
def test_full_size_executes_and_is_linear(pkg, fbp):
    """2048^2 kernels launch (shared-memory/launch limits) and stay linear; no oracle."""
    from paper_1608_03589_b200 import synth
    plan = pkg.get_plan(2048, 2048, 2048, None, None, (0.0, 1.0) if fbp else None)
    x = synth.config_batch(3 if fbp else 2, [0, 1], torch.device("cuda"))
    y = plan.execute(x)
    assert torch.isfinite(y).all() and y.abs().max() > 0
    y2 = plan.execute(torch.stack([x[1], 3.0 * x[0]]))
    assert torch.equal(y2[0], y[1])
    assert O.relative_l2(y2[1].cpu().numpy(), 3.0 * y[0].cpu().numpy()) < 1e-6
    assert torch.count_nonzero(plan.execute(torch.zeros_like(x))) == 0


def test_volume_reconstructor_shards_match_single_plan(pkg):
    """Slice-sharded multi-plan execution (here: three plans on one GPU, one host
    thread each) is bitwise identical to one plan over the whole volume."""
    vol = np.stack([phantoms.config_sinogram(1, i) for i in range(7)])
    ref = pkg.get_plan(512, 512, 512, None, None, (0.0, 1.0)).execute(dev(vol)).cpu().numpy()
    vr = pkg.VolumeReconstructor(512, 512, 512, filter_spec=(0.0, 1.0), devices=[0, 0, 0], chunk=2)
    out = vr.run(vol)
    assert np.array_equal(out, ref)
    assert pkg.shard_bounds(7, 3) == [(0, 2), (2, 4), (4, 7)]


@pytest.mark.parametrize("n", [2, 3, 5, 64, 129])
def test_small_and_odd_outputs(pkg, golden, n):
    z = golden("cfg0.npz")
    g = pkg.Sinogram(256, 256, z["sino"].astype(np.float64))
    ref = O.logpolar_backproject(z["sino"].astype(np.float64), n)
    assert report(f"bp n={n}", pkg.logpolar_backproject(g, n).values, ref) <= RTOL


def test_thin_annulus_and_all_fovea(pkg, golden):
    """Explicit rho0 close to 0: only pixels with ln r >= rho0 are non-zero (exact predicate)."""
    z = golden("cfg0.npz")
    gd = z["sino"].astype(np.float64)
    g = pkg.Sinogram(256, 256, gd)
    o = pkg.LogPolarOptions(rho0=-0.1, nrho=40)
    ref = O.logpolar_backproject(gd, 256, rho0=-0.1, nrho=40)
    got = pkg.logpolar_backproject(g, 256, o).values
    assert np.array_equal(got == 0, ref == 0)
    assert report("thin annulus", got, ref) <= RTOL


def test_empty_batch_and_stage_api_full_size(pkg):
    plan = pkg.get_plan(2048, 2048, 2048, None, None, None)
    out = plan.execute(torch.empty((0, 2048, 2048), device="cuda"))
    assert out.shape == (0, 2048, 2048)
    s = phantoms.config_sinogram(2, 7)
    lp = plan.logpolar(dev(s)[None])[0].cpu().numpy()
    ref = O.logpolar_stage(s.astype(np.float64), 2048)
    assert report("cfg2 logpolar stage", lp, ref) <= RTOL


@pytest.mark.parametrize("nt,nth", [(1100, 256), (1536, 256)])
def test_ramp_filter_both_m4096_kernels(pkg, nt, nth):
    """M = 4096 filters take the persistent TMA kernel when nt % 256 == 0 (1536) and the
    smem tile kernel otherwise (1100); both must match filter_sinogram (filtering.py:54-70)."""
    g = phantoms.sinogram(2200 + nt, nt, nth, 12, 0.05, 0.35, 0.01).astype(np.float64)
    s = pkg.Sinogram(nt, nth, g)
    got = pkg.filter_sinogram(s, pkg.FilterSpec()).values
    ref = O.ramp_filter(g, 0.0, 1.0)
    assert report(f"ramp M=4096 nt={nt}", got, ref) <= RTOL
    img = pkg.fbp(s, pkg.FilterSpec(), engine="logpolar", n=128).values
    assert report(f"fbp nt={nt}", img, O.fbp_logpolar(g, 128)) <= RTOL


@pytest.mark.parametrize("nt,n,fbp", [(256, 256, False), (256, 255, True), (512, 300, True), (2048, 2048, True)])
def test_no_out_of_bounds_writes(pkg, nt, n, fbp):
    """compute-sanitizer is unavailable on this pool: carve input, output and
    workspace out of one NaN-filled buffer with guard zones and check that every
    guard element survives a full execute (all kernels, TMA paths included)."""
    plan = pkg.get_plan(nt, nt, n, None, None, (0.0, 1.0) if fbp else None)
    b = 3
    guard = 1 << 16  # floats
    n_in, n_out = b * nt * nt, b * n * n
    ws_floats = (plan.workspace_bytes(2) + 3) // 4
    up = lambda v: (v + 63) // 64 * 64  # noqa: E731  (256-byte aligned carve-outs: the ABI's contract)
    o_in = guard
    o_out = up(o_in + n_in + guard)
    o_ws = up(o_out + n_out + guard)
    total = o_ws + ws_floats + guard
    big = torch.full((total,), float("nan"), device="cuda")
    x = pkg.synth.config_batch(3 if nt == 2048 else 0 if nt == 256 else 1, range(b), torch.device("cuda"))
    big[o_in:o_in + n_in] = x.reshape(-1)
    sino = big[o_in:o_in + n_in].view(b, nt, nt)
    out = big[o_out:o_out + n_out].view(b, n, n)
    ws = big[o_ws:o_ws + ws_floats].view(torch.uint8)
    plan.execute(sino, out=out, workspace=ws)
    torch.cuda.synchronize()
    for lo, hi in ((0, o_in), (o_in + n_in, o_out), (o_out + n_out, o_ws), (o_ws + ws_floats, total)):
        assert torch.isnan(big[lo:hi]).all(), f"guard [{lo},{hi}) overwritten"
    assert torch.equal(big[o_in:o_in + n_in], x.reshape(-1))  # input untouched
    assert torch.isfinite(out).all()
    ref = plan.execute(x)
    assert torch.equal(out, ref)
    with pytest.raises(ValueError, match="256-byte aligned"):
        plan.execute(sino, out=out, workspace=big[o_ws + 1:o_ws + 1 + ws_floats].view(torch.uint8))


@pytest.mark.parametrize("nt,nth,n", [(128, 90, 64), (256, 180, 128), (200, 96, 100), (512, 360, 256)])
def test_generic_sizes_vs_oracle(pkg, nt, nth, n):
    """Non-power-of-two angle counts (the reference's own examples use 90/180) run
    the Bluestein path; BP and FBP match the oracle."""
    rng = np.random.default_rng(nt + nth)
    gd = np.cumsum(rng.standard_normal((nt, nth)), axis=0).astype(np.float32).astype(np.float64) * 0.05
    g = pkg.Sinogram(nt, nth, gd)
    assert report(f"generic bp {nt}x{nth}->{n}", pkg.logpolar_backproject(g, n).values,
                  O.logpolar_backproject(gd, n)) <= RTOL
    assert report(f"generic fbp {nt}x{nth}->{n}", pkg.fbp(g, pkg.FilterSpec(), engine="logpolar", n=n).values,
                  O.fbp_logpolar(gd, n)) <= RTOL
    assert report(f"generic filter {nt}x{nth}", pkg.filter_sinogram(g, pkg.FilterSpec(lam=0.01)).values,
                  O.ramp_filter(gd, 0.01)) <= 1e-5


def test_reference_known_answers_on_device(pkg):
    """scratch_lp.py known answers (constant sinogram, pinned in tests/golden/kat.json)
    reproduced by the device path: interior means 3.05565 and 3.09808."""
    import json
    import os
    from conftest import GOLDEN
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))
    for nt, nth, n in ((128, 90, 64), (256, 180, 128)):
        b = pkg.logpolar_backproject(pkg.Sinogram(nt, nth, np.ones((nt, nth))), n).values
        xs = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
        X, Y = np.meshgrid(xs, xs)
        R = np.hypot(X, Y)
        inner = (R > 2 * math.exp(pkg.adaptive_rho0(n, n))) & (R <= 0.8)
        got, want = b[inner].mean(), kat[f"const_mean_{nt}_{nth}_{n}"]
        print(f"const mean {nt}x{nth}->{n}: {got:.6f} (reference {want:.6f})")
        assert abs(got - want) < 1e-5 * abs(want)


@pytest.mark.parametrize("nt,nth,n", [(128, 90, 64), (256, 180, 128)])
def test_spec_fovea_excluded_equivalence_with_naive(pkg, nt, nth, n):
    """log-polar vs the direct engine within 8e-2 relative L2 outside ||x|| <= 2 e^{rho0}
    (seeded ellipse phantoms stand in for the SPEC's Shepp-Logan)."""
    g = phantoms.sinogram(1200 + n, nt, nth, 10, 0.05, 0.35, 0.0)
    t = torch.from_numpy(g).cuda()[None]
    lp = pkg.logpolar_backproject_batch(t, n)[0].double().cpu().numpy()
    nv = pkg.naive_backproject(t, n)[0].double().cpu().numpy()
    xs = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
    R = np.hypot(*np.meshgrid(xs, xs))
    m = (R > 2 * math.exp(O.adaptive_rho0(n, n))) & (R <= 1.0)
    gap = float(np.linalg.norm(lp[m] - nv[m]) / np.linalg.norm(nv[m]))
    print(f"fovea-excluded LP vs naive {n}: {gap:.3e}")
    assert gap <= 8e-2


def test_spec_single_sector_reproduces_logpolar(pkg):
    """one sector covering everything with a_r = 1/4 reproduces logpolar_backproject
    within 5e-2 relative L2 away from the fovea."""
    n = 128
    g = phantoms.sinogram(1300, 256, 180, 10, 0.05, 0.35, 0.0).astype(np.float64)
    s = pkg.Sinogram(256, 180, g)
    pb = pkg.partial_backproject(s, [(0.0, math.pi / 2, 0.25)], n).values
    lp = pkg.logpolar_backproject(s, n).values
    xs = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
    R = np.hypot(*np.meshgrid(xs, xs))
    m = (R > 2 * math.exp(O.adaptive_rho0(n, n))) & (R <= 1.0)
    gap = float(np.linalg.norm(pb[m] - lp[m]) / np.linalg.norm(lp[m]))
    print(f"single sector vs logpolar: {gap:.3e}")
    assert gap <= 5e-2


_TMEM_AB = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1608_03589_b200 as p
from oracle import phantoms
g = torch.stack([torch.from_numpy(phantoms.config_sinogram(3, i)) for i in (0, 7)]).cuda()
plan = p.get_plan(2048, 2048, 2048, None, None, (0.0, 1.0))
np.save(sys.argv[2], plan.execute(g, chunk=2).cpu().numpy())
"""


def test_rho_conv_tmem_operands_bitwise(tmp_path):
    """K3 holds its loop invariants (K-hat column, first-pass taps, row-mix taps) in TMEM by default;
    LPBP_K3_TMEM=0 reads them from L2 / shared memory each slice.  Same arithmetic, so the two
    2048^2 FBP outputs are bitwise equal (each run in its own process: the switch is read once)."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for v in ("1", "0"):
        f = str(tmp_path / f"k3_tmem_{v}.npy")
        env = dict(os.environ, LPBP_K3_TMEM=v)
        r = subprocess.run([sys.executable, "-c", _TMEM_AB, repo, f], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    assert np.isfinite(outs[0]).all() and np.abs(outs[0]).max() > 0
    assert np.array_equal(outs[0], outs[1])


_K2P_AB = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1608_03589_b200 as p
from oracle import phantoms
out = {}
g = torch.stack([torch.from_numpy(phantoms.config_sinogram(3, i)) for i in (0, 7, 9)]).cuda()
plan = p.get_plan(2048, 2048, 2048, None, None, (0.0, 1.0))
out["p_rows_2048"] = np.int32(plan.info["p_rows"])
out["fbp2048"] = plan.execute(g, chunk=2).cpu().numpy()
out["lp2048"] = plan.logpolar(g[:1]).cpu().numpy()
g = torch.stack([torch.from_numpy(phantoms.config_sinogram(1, i)) for i in range(5)]).cuda()
out["fbp512"] = p.get_plan(512, 512, 512, None, None, (0.0, 1.0)).execute(g, chunk=3).cpu().numpy()
g = torch.from_numpy(phantoms.config_sinogram(0, 0))[None].cuda()
out["bp256"] = p.get_plan(256, 256, 256, None, None, None).execute(g).cpu().numpy()
torch.manual_seed(5)
g = torch.randn(3, 96, 1280, device="cuda").cumsum(1) * 0.05     # mixed-radix row DFTs (nphi = 5 x 512)
plan = p.get_plan(96, 1280, 64, None, None, (0.0, 1.0))
out["p_rows_mixed"] = np.int32(plan.info["p_rows"])
out["fbp_mixed"] = plan.execute(g, chunk=2).cpu().numpy()
np.savez(sys.argv[2], **out)
"""


def test_k2p_matches_frequency_domain_row_mix(tmp_path):
    """Default: K2p transforms the semi-polar rows and K3 takes their spectra as they are (p_rows = 1).
    LPBP_K2P=0: K2's nt row spectra and K3's frequency-domain row mix.  The two orders of the same
    linear maps agree to fp32 rounding at 256^2, 512^2 and 2048^2 (images and the log-polar stage) and on a
    mixed-radix plan (k_row_rdft_mixed_p against k_row_rdft_mixed + the row mix);
    each run in its own process (the switch is read once)."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for tag, extra in (("k2p1", {"LPBP_K2P": "1"}), ("k2p0", {"LPBP_K2P": "0"}), ("ycp0", {"LPBP_YCOMPACT": "0"})):
        f = str(tmp_path / f"{tag}.npz")
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, "-c", _K2P_AB, repo, f], env=env, capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    # LPBP_YCOMPACT=0 leaves the convolved spectra's rows in place instead of packing the needed bands back
    # to back: the same arithmetic on the same values, so every output is bitwise the default's
    for k in ("fbp2048", "lp2048", "fbp512", "bp256", "fbp_mixed"):
        assert np.array_equal(outs[0][k], outs[2][k]), k
    assert int(outs[0]["p_rows_2048"]) == 1 and int(outs[1]["p_rows_2048"]) == 0
    assert int(outs[0]["p_rows_mixed"]) == 1 and int(outs[1]["p_rows_mixed"]) == 0
    for k in ("fbp2048", "lp2048", "fbp512", "bp256", "fbp_mixed"):
        a, b = outs[0][k], outs[1][k]
        assert np.isfinite(a).all() and np.abs(a).max() > 0
        e = O.relative_l2(a, b)
        print(f"K2p vs row-mix path {k}: {e:.3e}")
        assert e <= 3e-6


@pytest.mark.parametrize("nth", [768, 1280, 1536, 2304, 2560, 3200, 3840])
def test_mixed_radix_row_dfts_vs_oracle(pkg, nth):
    """Angle counts whose nphi = 2 ntheta is Q x 2^k (Q = 3, 5, 9, 15, 25) take the mixed-radix
    row DFTs (mixed.cuh) in both directions; BP and FBP against the oracle, and the row spectra
    stage against numpy's rfft of the (filtered) rows."""
    nt, n = 96, 64
    q = 2 * nth
    while q % 2 == 0:
        q //= 2
    rng = np.random.default_rng(nth)
    gd = np.cumsum(rng.standard_normal((nt, nth)), axis=0).astype(np.float32).astype(np.float64) * 0.05
    plan = pkg.get_plan(nt, nth, n, None, None, (0.0, 1.0))
    assert plan.info["generic"] == 1 and plan.info["phi_q"] == q
    g = pkg.Sinogram(nt, nth, gd)
    assert report(f"mixed bp {nt}x{nth}->{n}", pkg.logpolar_backproject(g, n).values,
                  O.logpolar_backproject(gd, n)) <= RTOL
    assert report(f"mixed fbp {nt}x{nth}->{n}", pkg.fbp(g, pkg.FilterSpec(), engine="logpolar", n=n).values,
                  O.fbp_logpolar(gd, n)) <= RTOL


@pytest.mark.parametrize("nt,nth,n,fbp", [(96, 3200, 64, True), (96, 768, 64, False), (130, 1280, 100, True)])
def test_no_out_of_bounds_writes_mixed(pkg, nt, nth, n, fbp):
    """Guard zones (NaN) around input, output and workspace for the mixed-radix row DFTs and the
    unfused generic path (odd ntheta multiples, odd-looking nt), as test_no_out_of_bounds_writes does
    for the power-of-two path."""
    plan = pkg.get_plan(nt, nth, n, None, None, (0.0, 1.0) if fbp else None)
    assert plan.info["phi_q"] > 0
    b = 3
    guard = 1 << 16
    n_in, n_out = b * nt * nth, b * n * n
    ws_floats = (plan.workspace_bytes(2) + 3) // 4
    up = lambda v: (v + 63) // 64 * 64  # noqa: E731
    o_in = guard
    o_out = up(o_in + n_in + guard)
    o_ws = up(o_out + n_out + guard)
    total = o_ws + ws_floats + guard
    big = torch.full((total,), float("nan"), device="cuda")
    x = torch.randn(b, nt, nth, device="cuda")
    big[o_in:o_in + n_in] = x.reshape(-1)
    sino = big[o_in:o_in + n_in].view(b, nt, nth)
    out = big[o_out:o_out + n_out].view(b, n, n)
    ws = big[o_ws:o_ws + ws_floats].view(torch.uint8)
    plan.execute(sino, out=out, workspace=ws, chunk=2)
    torch.cuda.synchronize()
    for lo, hi in ((0, o_in), (o_in + n_in, o_out), (o_out + n_out, o_ws), (o_ws + ws_floats, total)):
        assert torch.isnan(big[lo:hi]).all(), f"guard [{lo},{hi}) overwritten"
    assert torch.isfinite(out).all()
    assert torch.equal(out, plan.execute(x, chunk=2))


@pytest.mark.parametrize("nt,nth,n", [(96, 3200, 64), (128, 768, 100)])
def test_mixed_fused_batch_invariance(pkg, nt, nth, n):
    """The fused mixed-radix inverse DFT + readout (bands of two rows, work units taken dynamically)
    gives bitwise the same images for any chunking of the batch, and the stage API's full log-polar
    image read out by the standalone readout agrees with it to fp32 rounding."""
    plan = pkg.get_plan(nt, nth, n, None, None, (0.0, 1.0))
    assert plan.info["phi_q"] > 0 and plan.info["band_rows"] == 2
    x = torch.randn(5, nt, nth, device="cuda")
    a = plan.execute(x, chunk=5)
    assert torch.equal(a, plan.execute(x, chunk=2))
    assert torch.equal(a, torch.cat([plan.execute(x[i:i + 1]) for i in range(5)]))
    lp = plan.logpolar(plan.filter(x))
    b = plan.readout(lp)
    assert O.relative_l2(b.cpu().numpy(), a.cpu().numpy()) < 1e-6


@pytest.mark.parametrize("nt,nth,n,fbp", [(97, 1280, 64, True), (131, 3200, 90, False), (64, 2304, 33, True)])
def test_mixed_radix_odd_and_small_shapes(pkg, nt, nth, n, fbp):
    """Mixed-radix angle counts with odd nt (row-spectra pitch padded to even), odd n and a small
    image: BP / FBP against the oracle."""
    rng = np.random.default_rng(nt * 7 + nth)
    gd = np.cumsum(rng.standard_normal((nt, nth)), axis=0).astype(np.float32).astype(np.float64) * 0.05
    g = pkg.Sinogram(nt, nth, gd)
    if fbp:
        got = pkg.fbp(g, pkg.FilterSpec(), engine="logpolar", n=n).values
        ref = O.fbp_logpolar(gd, n)
    else:
        got = pkg.logpolar_backproject(g, n).values
        ref = O.logpolar_backproject(gd, n)
    assert report(f"mixed odd {nt}x{nth}->{n} fbp={fbp}", got, ref) <= RTOL
