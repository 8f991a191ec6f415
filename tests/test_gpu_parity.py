"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (north_star): alpha/beta bit-exact; guarded output within 0.05 grey levels
(0-255 scale) of the fp64/__float128 oracle on every compared pixel.  Inputs are
the seeded workload generators (workloads/); the oracle never sees GPU output.
"""
import numpy as np
import pytest

import workloads
from parity import compare_guarded, compare_literal, grey_scale, psnr, TOL_GREY

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1811_02308_b200 import build

    build.build()
    import paper_1811_02308_b200 as fb

    return fb


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def _run(fb, w, flags=0, diag=False):
    import torch

    B, H, W = w.img.shape
    plan = fb.Plan(B, H, W, flags)
    img, th, sg = _dev(w.img), _dev(w.theta), _dev(w.sigma)
    if diag:
        out, d = fb.filter_diag(plan, img, th, sg, w.rho, w.N)
        torch.cuda.synchronize()
        return out.cpu().numpy(), {k: v.cpu().numpy() for k, v in d.items()}, plan
    out = fb.filter(plan, img, th, sg, w.rho, w.N)
    torch.cuda.synchronize()
    return out.cpu().numpy(), None, plan


# ------------------------------------------------------------------ step a1
@pytest.mark.parametrize("shape,rho", [
    ((1, 1, 1), 0), ((1, 7, 7), 3), ((2, 37, 53), 5), ((1, 64, 300), 20), ((1, 300, 41), 20),
    ((3, 97, 129), 2), ((1, 200, 333), 40), ((1, 193, 517), 96), ((1, 256, 256), 0),
    # width % 4 == 0: interior tiles staged by TMA from a 16-byte aligned column
    ((1, 256, 256), 9), ((1, 192, 320), 10), ((2, 200, 260), 11), ((1, 300, 512), 24),
    ((1, 260, 388), 33)])
def test_bounds_bit_exact(fb, orc, shape, rho):
    import torch

    rng = np.random.default_rng(sum(shape) * 31 + rho)
    f = rng.normal(100, 60, shape).astype(np.float32)  # non-integer, negative values too
    plan = fb.Plan(*shape)
    a, b = fb.bounds(plan, _dev(f), rho)
    torch.cuda.synchronize()
    ra, rb = orc.bounds(f, rho)
    assert np.array_equal(a.cpu().numpy(), ra)
    assert np.array_equal(b.cpu().numpy(), rb)


def test_bounds_full_4k_bit_exact(fb, orc):
    import torch

    w = workloads.config(4)
    plan = fb.Plan(*w.shape)
    a, b = fb.bounds(plan, _dev(w.img), w.rho)
    torch.cuda.synchronize()
    ra, rb = orc.bounds(w.img, w.rho)  # exhaustive 41x41 scan, all 8.3 Mpx
    assert np.array_equal(a.cpu().numpy(), ra) and np.array_equal(b.cpu().numpy(), rb)


# ------------------------------------------------------------------ whole path, configs
@pytest.mark.parametrize("cfg", [1, 2])
def test_config_full_size_all_pixels(fb, orc, cfg):
    w = workloads.config(cfg)
    out, d, plan = _run(fb, w, diag=True)
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    mx, nbad, _ = compare_guarded(out, o, 1.0)
    assert nbad == 0, f"max |delta| = {mx} grey"
    # bounds reported by the diag path are bit-exact
    ra, rb = orc.bounds(w.img, w.rho)
    assert np.array_equal(d["alpha"], ra) and np.array_equal(d["beta"], rb)


@pytest.mark.parametrize("cfg,scale", [(3, 0.3), (4, 0.2)])
def test_config_scaled_all_pixels(fb, orc, cfg, scale):
    w = workloads.config(cfg, scale=scale)
    out, _, _ = _run(fb, w)
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    mx, nbad, _ = compare_guarded(out, o, 1.0)
    assert nbad == 0, f"max |delta| = {mx} grey"


@pytest.mark.parametrize("gen,rho,N", [("texture", 2, 10), ("rectangles", 2, 10), ("rectangles", 20, 10),
                                       ("rectangles", 40, 4), ("texture", 10, 6)])
def test_config5_cell_all_pixels(fb, orc, gen, rho, N):
    """Config-5 (rho, N) cells on one 384^2 image of each generator, every pixel.
    High-kappa pixels here (up to ~900) exposed fp32 rounding of lambda and t0
    (amplified by kappa), which is why C2 derives them in fp64."""
    w = workloads.config5(rho, N, batch=1, size=384, generator=gen)
    out, _, _ = _run(fb, w)
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    mx, nbad, _ = compare_guarded(out, o, 1.0)
    assert nbad == 0, f"max |delta| = {mx} grey"


@pytest.mark.parametrize("cfg,nsample", [(3, 3000), (4, 1500)])
def test_config_full_size_sampled(fb, orc, cfg, nsample):
    """Full BASELINE sizes, same launch configuration as bench.py; oracle on a
    seeded sample of pixels (plus the four corners and edge midpoints)."""
    w = workloads.config(cfg)
    out, d, plan = _run(fb, w, diag=True)
    B, H, W = w.shape
    rng = np.random.default_rng(cfg)
    idx = rng.choice(w.img.size, nsample, replace=False)
    edges = [0, W - 1, (H - 1) * W, H * W - 1, W // 2, (H // 2) * W, (H // 2) * W + W - 1, (H - 1) * W + W // 2]
    idx = np.unique(np.concatenate([idx, edges]))
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N, pixels=idx)
    mx, nbad, _ = compare_guarded(out.ravel()[idx], o, 1.0)
    assert nbad == 0, f"max |delta| = {mx} grey"
    # properties that hold at any size: g-hat inside [alpha, beta] wherever the
    # guard did not fire and kappa is moderate is not guaranteed (reading R7),
    # but it is finite everywhere and identity pixels copy f exactly
    assert np.all(np.isfinite(out))
    ident = (d["code"] & fb.CODE_IDENTITY) > 0
    assert np.array_equal(out[ident], w.img[ident])


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("N", list(range(0, 11)))
@pytest.mark.parametrize("rho,fused", [(4, False), (13, False), (13, True)])
def test_every_degree(fb, orc, N, rho, fused):
    w = workloads.random_case(2, 45, 61, seed=100 + N, kind="rect", rho=rho, N=N)
    out, _, _ = _run(fb, w, flags=fb.FLAG_FUSED if fused else 0)
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    mx, nbad, _ = compare_guarded(out, o, 1.0)
    assert nbad == 0, f"N={N}: max |delta| = {mx}"


@pytest.mark.parametrize("rho,N", [(10, 9), (10, 10), (20, 10), (40, 6)])
def test_wide_windows_high_degree(fb, orc, rho, N):
    """Prefix-row widths E = 11 / 13 with N = 9, 10 run with one pixel per
    thread per step (shared-memory-driven PPT choice); texture content."""
    w = workloads.random_case(1, 120, 300, seed=300 + rho + N, kind="texture", rho=rho, N=N)
    out, _, _ = _run(fb, w)
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    mx, nbad, _ = compare_guarded(out, o, 1.0)
    assert nbad == 0, f"rho={rho} N={N}: max |delta| = {mx}"


@pytest.mark.parametrize("kind,shape,rho,N", [
    ("rect", (1, 7, 7), 3, 5),          # window == image
    ("rect", (1, 1, 1), 0, 4),          # single pixel
    ("rect", (1, 5, 300), 2, 6),        # 2rho+1 == H
    ("texture", (1, 131, 257), 5, 8),   # ragged tails in both directions
    ("voronoi", (2, 150, 140), 12, 8),
    ("uniform", (1, 66, 70), 1, 3),
    ("float", (1, 57, 91), 3, 6),       # non-integer, negative, other scale
    ("flat", (1, 40, 40), 3, 5),        # identity pixels
    ("texture", (1, 96, 200), 40, 8),   # rho = 40 (config 5's largest)
    ("rect", (1, 200, 230), 96, 4),     # largest supported rho
])
@pytest.mark.parametrize("fused", [False, True])
def test_edge_shapes(fb, orc, kind, shape, rho, N, fused):
    """Both bounds placements (FABF_FLAG_FUSED: alpha, beta from k_filter's own
    van Herk / Gil-Werman passes, reported by the diag path and bit-exact)."""
    w = workloads.random_case(*shape, seed=7, kind=kind, rho=rho, N=N)
    out, d, _ = _run(fb, w, flags=fb.FLAG_FUSED if fused else 0, diag=True)
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    sc = grey_scale(w.img)
    mx, nbad, _ = compare_guarded(out, o, sc)
    assert nbad == 0, f"max |delta| = {mx} grey"
    ident = (o["code"] & 1) > 0
    assert np.array_equal(out[ident], w.img[ident])
    assert np.array_equal((d["code"] & 1) > 0, ident)
    ra, rb = orc.bounds(w.img, w.rho)
    assert np.array_equal(d["alpha"], ra) and np.array_equal(d["beta"], rb)


@pytest.mark.parametrize("kind,shape,rho,N", [
    ("cfg1", None, 3, 5), ("cfg2", None, 5, 6),
    ("rect", (1, 5, 300), 2, 6), ("texture", (1, 131, 257), 5, 8), ("rect", (2, 37, 53), 4, 10),
    ("rect", (1, 7, 7), 3, 5), ("rect", (1, 1, 1), 0, 4), ("float", (1, 57, 91), 3, 6),
    ("flat", (1, 40, 40), 1, 5), ("voronoi", (1, 200, 260), 5, 4)])
def test_fused_small_rho_all_pixels(fb, orc, kind, shape, rho, N):
    """rho <= 5 without diagnostics: bounds computed inside k_filter (per-column
    ring + horizontal min/max, no k_bounds, no alpha/beta planes).  Every pixel
    against the oracle; identity pixels copy f bit-exactly."""
    if kind == "cfg1":
        w = workloads.config(1)
    elif kind == "cfg2":
        w = workloads.config(2)
    else:
        w = workloads.random_case(*shape, seed=11, kind=kind, rho=rho, N=N)
    out, _, _ = _run(fb, w)
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    mx, nbad, _ = compare_guarded(out, o, grey_scale(w.img))
    assert nbad == 0, f"max |delta| = {mx} grey"
    ident = (o["code"] & 1) > 0
    assert np.array_equal(out[ident], w.img[ident])


def test_rho0_is_exact_copy(fb):
    w = workloads.random_case(2, 33, 17, seed=3, rho=0, N=5)
    out, _, _ = _run(fb, w)
    assert np.array_equal(out, w.img)


def test_literal_and_clamp_flags(fb, orc):
    w = workloads.config(4, scale=0.1)
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    out_l, _, _ = _run(fb, w, flags=fb.FLAG_LITERAL)
    mx, nbad, nexcl = compare_literal(out_l, o, 1.0)
    assert nbad == 0, f"literal max |delta| = {mx} ({nexcl} ill-conditioned pixels excluded)"
    out_c, d, _ = _run(fb, w, flags=fb.FLAG_CLAMP, diag=True)
    ra, rb = orc.bounds(w.img, w.rho)
    assert np.all(out_c >= ra) and np.all(out_c <= rb)
    ref = np.clip(o["g_guard"], ra, rb)
    assert np.max(np.abs(out_c - ref)) <= TOL_GREY


def test_extreme_range_parameters(fb, orc):
    """theta far outside [alpha, beta] (regimes A with |t0|>1 and C), tiny and
    huge sigma (lambda from 1e-9 to 1e6)."""
    rng = np.random.default_rng(17)
    w = workloads.random_case(1, 60, 80, seed=17, kind="rect", rho=3, N=6)
    th = w.theta.copy()
    sg = w.sigma.copy()
    th[0, :15] = w.img[0, :15] + rng.uniform(-600, 600, (15, 80))      # far theta
    th[0, 15:30] = w.img[0, 15:30] + rng.uniform(-150, 150, (15, 80))  # |t0| ~ 1..2
    sg[0, 30:40] = rng.uniform(0.3, 2.0, (10, 80))                      # huge lambda
    sg[0, 40:50] = rng.uniform(1e3, 1e5, (10, 80))                      # lambda -> 0
    w2 = workloads.Workload("extreme", w.img, th.astype(np.float32), sg.astype(np.float32), 3, 6)
    out, d, _ = _run(fb, w2, diag=True)
    o = orc.fast(w2.img, w2.theta, w2.sigma, 3, 6)
    fin = np.isfinite(o["g_guard"])
    mx, nbad, err = compare_guarded(out.ravel()[fin.ravel()], {k: v.ravel()[fin.ravel()] for k, v in o.items()}, 1.0)
    assert nbad == 0, f"max |delta| = {mx}"
    assert np.any(d["code"] & fb.CODE_FAR_THETA) and np.any(d["code"] & fb.CODE_SMALL_LAMBDA)


def test_fallback_path_parity(fb, orc):
    """A tile mixing a near-flat dark area with full-contrast texture: the
    centring amplification flag routes the flat windows to the exact-moment
    fallback; results must still match the oracle."""
    rng = np.random.default_rng(5)
    H, W = 96, 160
    f = np.rint(rng.uniform(0, 255, (H, W)))
    f[:, :60] = np.rint(3 + rng.uniform(0, 2, (H, 60)))  # range ~2 next to range ~255
    f = f.astype(np.float32)[None]
    th = (f + rng.uniform(-1, 1, f.shape)).astype(np.float32)
    sg = rng.uniform(0.5, 20, f.shape).astype(np.float32)
    w = workloads.Workload("fallback", f, th, sg, 2, 10)
    out, d, plan = _run(fb, w, diag=True)
    assert plan.last_fallback_count() > 0
    assert np.any(d["code"] & fb.CODE_FALLBACK)
    o = orc.fast(f, th, sg, 2, 10)
    mx, nbad, _ = compare_guarded(out, o, 1.0)
    assert nbad == 0, f"max |delta| = {mx}"


@pytest.mark.parametrize("rho,N,fused", [(2, 10, False), (12, 10, False), (40, 8, False), (12, 10, True)])
def test_fallback_segments_parity(fb, orc, rho, N, fused):
    """k_fallback_seg (the exact-moment fallback by 32-pixel row segments with
    their own centre, O(rho) per pixel) on a flat-next-to-texture image with a
    long fallback list, every pixel against the oracle; a second call on the
    same plan (the segment bitmap is cleared) gives the same result."""
    import torch

    rng = np.random.default_rng(50 + rho)
    H, W = max(120, 2 * rho + 40), 200
    f = np.rint(rng.uniform(0, 255, (H, W)))
    f[:, :90] = np.rint(3 + rng.uniform(0, 2, (H, 90)))
    f[H // 2:, 150:] = np.rint(250 + rng.uniform(0, 3, (H - H // 2, 50)))  # a second, bright flat area
    f = f.astype(np.float32)[None]
    th = (f + rng.uniform(-1, 1, f.shape)).astype(np.float32)
    sg = rng.uniform(0.5, 20, f.shape).astype(np.float32)
    plan = fb.Plan(*f.shape, fb.FLAG_FUSED if fused else 0)
    out = fb.filter(plan, _dev(f), _dev(th), _dev(sg), rho, N)
    torch.cuda.synchronize()
    nfb = plan.last_fallback_count()
    assert nfb > 0
    out2 = fb.filter(plan, _dev(f), _dev(th), _dev(sg), rho, N)
    torch.cuda.synchronize()
    assert torch.equal(out, out2) and plan.last_fallback_count() == nfb
    o = orc.fast(f, th, sg, rho, N)
    mx, nbad, _ = compare_guarded(out.cpu().numpy(), o, 1.0)
    assert nbad == 0, f"max |delta| = {mx} ({nfb} fallback pixels)"


def test_debug_flag_validates_preconditions(fb):
    """FABF_FLAG_DEBUG: the device-side check counts pixels with sigma <= 0 or
    a non-finite f / theta / sigma and reports the first one's flat index;
    clean inputs report (0, -1); the host entry point checks every band; a plan
    without the flag refuses the query."""
    import torch

    w = workloads.config(1, scale=0.5)
    B, H, W = w.shape
    plan = fb.Plan(B, H, W, fb.FLAG_DEBUG)
    img, th, sg = _dev(w.img), _dev(w.theta), _dev(w.sigma)
    out = fb.filter(plan, img, th, sg, w.rho, w.N)
    assert plan.debug_status() == (0, -1)
    ref = fb.filter(fb.Plan(B, H, W), img, th, sg, w.rho, w.N)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)  # the check does not change the result
    bad = {5 * W + 7: ("sigma", 0.0), 9 * W + 1: ("theta", float("nan")),
           (H - 1) * W + W - 1: ("sigma", -2.0), 3 * W + 100: ("img", float("inf"))}
    planes = {"img": w.img.copy(), "theta": w.theta.copy(), "sigma": w.sigma.copy()}
    for o, (name, v) in bad.items():
        planes[name].reshape(-1)[o] = v
    fb.filter(plan, _dev(planes["img"]), _dev(planes["theta"]), _dev(planes["sigma"]), w.rho, w.N)
    assert plan.debug_status() == (len(bad), min(bad))
    host_out = np.empty_like(w.img)
    fb.filter_host(plan, planes["img"], planes["theta"], planes["sigma"], w.rho, w.N, host_out)
    assert plan.debug_status() == (len(bad), min(bad))
    fb.filter(plan, img, th, sg, w.rho, w.N)  # a fresh word per call
    assert plan.debug_status() == (0, -1)
    with pytest.raises(fb.FabfError):
        fb.Plan(B, H, W).debug_status()


def test_filter_events_matches_filter(fb):
    """fabf_filter_events: same output as fabf_filter, five recorded events in
    kernel order with non-negative gaps (no host sync inside)."""
    import torch

    w = workloads.config(3, scale=0.25)
    plan = fb.Plan(*w.shape)
    img, th, sg = _dev(w.img), _dev(w.theta), _dev(w.sigma)
    ref = fb.filter(plan, img, th, sg, w.rho, w.N)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    for e in evs:
        e.record()
    out = fb.filter_events(plan, img, th, sg, w.rho, w.N, evs)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    gaps = [evs[i].elapsed_time(evs[i + 1]) for i in range(4)]
    assert all(g >= 0.0 for g in gaps) and gaps[0] > 0.0 and gaps[2] > 0.0


@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (3, 0.5), (4, 0.25)])
def test_host_entry_point_matches_oracle(fb, orc, cfg, scale):
    """fabf_filter_host (host buffers, row-band pipeline with copies on their own
    streams): alpha/beta-exact identity pixels, every pixel within tolerance of
    the oracle, and within 1e-3 grey of the device entry point (band edges move
    segment boundaries, hence the tile-local centring of the running sums)."""
    import torch

    w = workloads.config(cfg, scale=scale)
    plan = fb.Plan(*w.shape)
    dev = fb.filter(plan, _dev(w.img), _dev(w.theta), _dev(w.sigma), w.rho, w.N)
    torch.cuda.synchronize()
    host_out = np.empty_like(w.img)
    fb.filter_host(plan, w.img, w.theta, w.sigma, w.rho, w.N, host_out)
    assert np.max(np.abs(host_out.astype(np.float64) - dev.cpu().numpy())) <= 1e-3
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    mx, nbad, _ = compare_guarded(host_out, o, 1.0)
    assert nbad == 0, f"max |delta| = {mx} grey"
    # a second call reuses the staging buffers and the copy streams
    host2 = np.empty_like(w.img)
    fb.filter_host(plan, w.img, w.theta, w.sigma, w.rho, w.N, host2)
    assert np.array_equal(host2, host_out)


@pytest.mark.parametrize("B,H,W,rho,N", [(3, 300, 260, 4, 6), (3, 300, 260, 12, 8),
                                         # last band a single row (H = 9 * 64 + 1), rho 40
                                         (1, 577, 200, 40, 6),
                                         # rho + 1 > 64: bands of two tiles or more
                                         (2, 420, 150, 70, 4)])
def test_host_entry_point_batch(fb, orc, B, H, W, rho, N):
    """fabf_filter_host on batches and band-partition edge cases (bands per
    frame, fused and unfused bounds, a one-row last band, halos wider than a
    tile): every pixel against the oracle."""
    w = workloads.random_case(B, H, W, seed=77 + rho, kind="voronoi", rho=rho, N=N)
    plan = fb.Plan(*w.shape)
    host_out = np.empty_like(w.img)
    fb.filter_host(plan, w.img, w.theta, w.sigma, w.rho, w.N, host_out)
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    mx, nbad, _ = compare_guarded(host_out, o, 1.0)
    assert nbad == 0, f"max |delta| = {mx} grey"


@pytest.mark.parametrize("cfg", [1, 3])
def test_cuda_graph_capture_and_replay(fb, cfg):
    """fabf_filter is graph-capturable (include/fabf.h): capture one call on a
    side stream, replay it, and get the eager result bit-exactly (fused and
    separate-bounds paths)."""
    import torch

    w = workloads.config(cfg, scale=0.5)
    plan = fb.Plan(*w.shape)
    img, th, sg = _dev(w.img), _dev(w.theta), _dev(w.sigma)
    ref = fb.filter(plan, img, th, sg, w.rho, w.N)
    out = torch.empty_like(img)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fb.filter(plan, img, th, sg, w.rho, w.N, out=out)  # warm-up on the capture stream
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            fb.filter(plan, img, th, sg, w.rho, w.N, out=out, stream=s)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_deterministic_and_stream_safe(fb):
    import torch

    w = workloads.config(2)
    plan = fb.Plan(*w.shape)
    img, th, sg = _dev(w.img), _dev(w.theta), _dev(w.sigma)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a = fb.filter(plan, img, th, sg, w.rho, w.N)
        b = fb.filter(plan, img, th, sg, w.rho, w.N)
    s.synchronize()
    assert torch.equal(a, b)


def test_argument_errors(fb):
    import torch

    plan = fb.Plan(1, 16, 16)
    x = torch.zeros(1, 16, 16, device="cuda")
    with pytest.raises(fb.FabfError) as e:
        fb.filter(plan, x, x, x, 8, 3)  # 2rho+1 > 16
    assert e.value.status == 1
    with pytest.raises(fb.FabfError) as e:
        fb.filter(plan, x, x, x, 2, 11)  # N > FABF_MAX_N
    assert e.value.status == 2
    with pytest.raises(fb.FabfError) as e:
        fb.filter(plan, x, x, x, 2, 3, out=x)  # out overlaps inputs
    assert e.value.status == 1
    with pytest.raises(fb.FabfError):
        fb.filter(plan, x, x, x, -1, 3)


def test_psnr_against_brute_force_config1(fb, orc):
    w = workloads.config(1)
    out, _, _ = _run(fb, w)
    g = orc.brute(w.img, w.theta, w.sigma, w.rho)
    assert psnr(out, g) > 40.0  # the paper's acceptance bar


@pytest.mark.parametrize("B,H,W,C,rho,N", [(2, 96, 130, 3, 5, 6), (1, 120, 200, 3, 12, 8), (1, 37, 53, 3, 3, 5),
                                           (1, 64, 64, 4, 2, 4)])
def test_colour_interleaved_channel_by_channel(fb, orc, B, H, W, C, rho, N):
    """NEXT-3 colour (channel by channel): fabf_filter_interleaved on
    B x H x W x C interleaved buffers equals the oracle applied to each channel
    plane (different content per channel); odd pixel counts included."""
    import torch

    rng = np.random.default_rng(B * 1000 + H + C)
    kinds = ["rect", "texture", "voronoi", "float"]
    planes = [workloads.random_case(B, H, W, seed=40 + ch, kind=kinds[ch % 4], rho=rho, N=N) for ch in range(C)]
    img = np.stack([p.img for p in planes], axis=-1).astype(np.float32)
    th = np.stack([p.theta for p in planes], axis=-1).astype(np.float32)
    sg = np.stack([p.sigma for p in planes], axis=-1).astype(np.float32)
    plan = fb.Plan(B * C, H, W)
    out = fb.filter_interleaved(plan, _dev(img), _dev(th), _dev(sg), rho, N)
    torch.cuda.synchronize()
    out = out.cpu().numpy()
    assert out.shape == img.shape
    for ch in range(C):
        o = orc.fast(img[..., ch], th[..., ch], sg[..., ch], rho, N)
        mx, nbad, _ = compare_guarded(out[..., ch], o, grey_scale(img[..., ch]))
        assert nbad == 0, f"channel {ch}: max |delta| = {mx}"
    with pytest.raises(fb.FabfError):
        fb.filter_interleaved(fb.Plan(B * C + 1, H, W), _dev(img), _dev(th), _dev(sg), rho, N)


@pytest.mark.parametrize("kind,shape,rho", [("cfg1", None, 3), ("cfg2", None, 5), ("rect", (2, 70, 91), 10),
                                            ("float", (1, 57, 91), 3), ("flat", (1, 40, 40), 2),
                                            ("texture", (1, 150, 140), 60)])
def test_mozerov_baseline(fb, orc, kind, shape, rho):
    """NEXT-4: fabf_filter_mozerov (eq.(29) at N = 0 on [f, 2 fbar - f])
    against the oracle's __float128 version, every pixel (the rho = 60 case
    runs the 16 x 16 tile variant)."""
    import torch

    if kind == "cfg1":
        w = workloads.config(1)
    elif kind == "cfg2":
        w = workloads.config(2)
    else:
        w = workloads.random_case(*shape, seed=19, kind=kind, rho=rho, N=0)
    plan = fb.Plan(*w.shape)
    out = fb.filter_mozerov(plan, _dev(w.img), _dev(w.theta), _dev(w.sigma), rho)
    torch.cuda.synchronize()
    ref = orc.mozerov(w.img, w.theta, w.sigma, rho)
    sc = grey_scale(w.img)
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref) / sc
    assert err.max() <= TOL_GREY, f"max |delta| = {err.max()} grey"


@pytest.mark.parametrize("kind,shape,rho,N,prm", [
    ("voronoi", (1, 160, 200), 5, 5, {}),
    ("texture", (2, 97, 131), 3, 6, dict(log_scale=0.8, sigma_lo=6.0, sigma_hi=30.0, log_sat=10.0)),
    ("rect", (1, 120, 90), 12, 8, dict(log_scale=2.0, sigma_lo=12.0, sigma_hi=45.0, log_sat=25.0))])
def test_sharpen_application(fb, orc, kind, shape, rho, N, prm):
    """NEXT-2: the device maps equal the oracle's (theta to fp32
    rounding of the box mean, sigma to fp32 LoG rounding), and the whole
    application (maps + Algorithm 1 from f alone) matches the oracle run on
    those maps, every pixel."""
    import torch

    w = workloads.random_case(*shape, seed=71, kind=kind, rho=rho, N=N)
    plan = fb.Plan(*w.shape)
    full = dict(fb.SHARPEN_DEFAULTS)
    full.update(prm)
    th, sg = fb.sharpen_maps(plan, _dev(w.img), rho, **prm)
    out = fb.filter_sharpen(plan, _dev(w.img), rho, N, **prm)
    torch.cuda.synchronize()
    th, sg, out = th.cpu().numpy(), sg.cpu().numpy(), out.cpu().numpy()
    rth, rsg = orc.sharpen_maps(w.img, rho, **full)
    assert np.max(np.abs(th - rth)) < 1e-3
    assert np.max(np.abs(sg - rsg)) < 1e-3
    assert sg.min() >= full["sigma_lo"] - 1e-4 and sg.max() <= full["sigma_hi"] + 1e-4
    o = orc.fast(w.img, th, sg, rho, N)
    mx, nbad, _ = compare_guarded(out, o, 1.0)
    assert nbad == 0, f"max |delta| = {mx} grey"
    assert plan.last_launch_count() >= 2


def test_row_band_subproblems_on_device(fb, orc):
    """SURVEY 8(e) row-band split, the per-rank computation on real kernels:
    each band plus rho halo rows of f (what shard.exchange_halo delivers),
    filtered as an image of its own and cropped, equals the oracle's rows of
    the whole frame -- three bands, the middle one with halos on both sides
    (the exchange itself is covered on CPU, tests/test_multi_gloo.py)."""
    import torch

    w = workloads.random_case(1, 150, 140, seed=97, kind="voronoi", rho=6, N=6)
    ref = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    sc = grey_scale(w.img)
    from paper_1811_02308_b200.shard import band_shard

    for rank in range(3):
        first, n = band_shard(150, 3, rank, rho=w.rho)
        lo, hi = max(0, first - w.rho), min(150, first + n + w.rho)
        top = first - lo
        f = np.ascontiguousarray(w.img[:, lo:hi])
        th, sg = f.copy(), np.ones_like(f)
        th[:, top:top + n] = w.theta[:, first:first + n]
        sg[:, top:top + n] = w.sigma[:, first:first + n]
        plan = fb.Plan(*f.shape)
        out = fb.filter(plan, _dev(f), _dev(th), _dev(sg), w.rho, w.N)
        torch.cuda.synchronize()
        part = {k: v[:, first:first + n] for k, v in ref.items()}
        mx, nbad, _ = compare_guarded(out.cpu().numpy()[:, top:top + n], part, sc)
        assert nbad == 0, f"band {rank}: max |delta| = {mx} grey"


@pytest.mark.parametrize("kind,shape,patch", [
    ("texture", (2, 97, 131), 3), ("rect", (1, 120, 90), 1), ("float", (1, 70, 75), 5), ("voronoi", (1, 33, 200), 16),
    ("flat", (1, 40, 40), 0), ("texture", (1, 20, 17), 2)])
def test_texture_maps(fb, orc, kind, shape, patch):
    """NEXT-2 (reading R19): the device mRTV / sigma maps equal the
    oracle's direct window scans, every pixel (the gradient magnitudes are the
    same fp64 values on both sides, so the window max is exact; the sums differ
    by their order only); ragged tiles, a window as wide as a tile, patch 0."""
    import torch

    w = workloads.random_case(*shape, seed=91 + patch, kind=kind, rho=2, N=2)
    plan = fb.Plan(*w.shape)
    prm = dict(patch=patch, sigma_lo=6.0, sigma_hi=44.0, mrtv_sat=9.0, eps=1e-3)
    sg, m = fb.texture_maps(plan, _dev(w.img), want_mrtv=True, **prm)
    torch.cuda.synchronize()
    rm, rsg = orc.texture_maps(w.img, **prm)
    sg, m = sg.cpu().numpy(), m.cpu().numpy()
    assert np.max(np.abs(m - rm.astype(np.float32))) <= 1e-5 * max(1.0, float(rm.max()))
    assert np.max(np.abs(sg - rsg)) <= 1e-4
    assert sg.min() >= 6.0 - 1e-5 and sg.max() <= 44.0 + 1e-5


def test_texture_entry_points_refuse_bad_arguments(fb):
    """fabf_texture_maps / fabf_filter_texture: INVALID_ARGUMENT for a patch
    outside [0, 16] or wider than the image, non-positive map parameters,
    sigma_hi < sigma_lo, and intermediates that overlap the input."""
    import torch

    plan = fb.Plan(1, 24, 40)
    img = torch.rand(1, 24, 40, device="cuda") * 255
    for bad in (dict(patch=17), dict(patch=-1), dict(patch=12), dict(mrtv_sat=0.0), dict(eps=0.0),
                dict(sigma_lo=0.0), dict(sigma_lo=9.0, sigma_hi=8.0), dict(second_scale=0.0)):
        with pytest.raises(fb.FabfError) as e:
            fb.texture_maps(plan, img, **bad)
        assert e.value.status == 1, bad
    with pytest.raises(fb.FabfError):
        fb.filter_texture(plan, img, 2, 3, pass1=img)
    with pytest.raises(fb.FabfError):
        fb.filter_texture(plan, img, 12, 3)  # window taller than the image
    with pytest.raises(fb.FabfError):
        fb.filter_texture(plan, img, 2, 3, rho_sharpen=12)
    out = fb.filter_texture(plan, img, 2, 3)  # the plan still works afterwards
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()


@pytest.mark.parametrize("kind,shape,rho,N,rs", [
    ("texture", (1, 150, 170), 5, 5, 3), ("rect", (2, 90, 110), 3, 6, 3), ("voronoi", (1, 128, 96), 10, 8, 5)])
def test_texture_application(fb, orc, kind, shape, rho, N, rs):
    """NEXT-2: Algorithm 1 three times.  Stage by stage -- every
    pass of the device pipeline against the oracle evaluated on the device's
    own previous intermediate (each stage's error, every pixel, within the
    0.05-grey bar) -- and end to end against the oracle's own pipeline."""
    import torch

    w = workloads.random_case(*shape, seed=95, kind=kind, rho=rho, N=N)
    plan = fb.Plan(*w.shape)
    tp = dict(fb.TEXTURE_DEFAULTS)
    tp.update(patch=2, sigma_hi=35.0)
    sp = dict(log_scale=1.0, sigma_lo=9.0, sigma_hi=25.0, log_sat=15.0)
    img = _dev(w.img)
    g1, g2 = torch.empty_like(img), torch.empty_like(img)
    out = fb.filter_texture(plan, img, rho, N, texture=tp, sharpen=sp, rho_sharpen=rs, pass1=g1, pass2=g2)
    launches = plan.last_launch_count()
    out_plain = fb.filter_texture(plan, img, rho, N, texture=tp, sharpen=sp, rho_sharpen=rs)  # plan-owned intermediates
    sg, _ = fb.texture_maps(plan, img, **tp)
    torch.cuda.synchronize()
    assert torch.equal(out, out_plain)
    assert launches >= 8  # 2 map kernels + 3 x (bounds or fused filter, fallback)
    sg, g1, g2, out = sg.cpu().numpy(), g1.cpu().numpy(), g2.cpu().numpy(), out.cpu().numpy()
    sc = grey_scale(w.img)
    o1 = orc.fast(w.img, w.img, sg, rho, N)
    mx, nbad, _ = compare_guarded(g1, o1, sc)
    assert nbad == 0, f"pass 1: max |delta| = {mx} grey"
    o2 = orc.fast(g1, g1, (np.float32(tp["second_scale"]) * sg).astype(np.float32), rho, N)
    mx, nbad, _ = compare_guarded(g2, o2, sc)
    assert nbad == 0, f"pass 2: max |delta| = {mx} grey"
    th3, sg3 = fb.sharpen_maps(plan, _dev(g2), rs, **sp)
    torch.cuda.synchronize()
    o3 = orc.fast(g2, th3.cpu().numpy(), sg3.cpu().numpy(), rs, N)
    mx, nbad, _ = compare_guarded(out, o3, sc)
    assert nbad == 0, f"pass 3: max |delta| = {mx} grey"
    # end to end: the oracle's own pipeline from f alone (errors of three passes compound)
    ref = orc.texture_pipeline(w.img, rho, N, texture=tp, sharpen=sp, rho_sharpen=rs)
    d = np.abs(out.astype(np.float64) - ref["out"]) / sc
    assert np.quantile(d, 0.999) <= TOL_GREY, f"end to end p99.9 = {np.quantile(d, 0.999)} grey, max {d.max()}"


def test_texture_application_colour_with_grey_map(fb, orc):
    """The paper's colour procedure: mRTV / sigma on the grey
    version, the channels filtered one by one with that map
    (fabf_filter_texture_map).  Stage by stage against the oracle on the
    device's own intermediates, and the map equals the oracle's map of the grey
    image."""
    import torch

    rho, N, rs = 4, 5, 3
    w = workloads.random_case(3, 90, 104, seed=99, kind="texture", rho=rho, N=N)  # three channel planes
    grey = w.img.mean(axis=0, keepdims=True).astype(np.float32)
    tp = dict(patch=2, sigma_lo=7.0, sigma_hi=32.0, mrtv_sat=10.0, eps=1e-3)
    sp = dict(log_scale=1.0, sigma_lo=9.0, sigma_hi=25.0, log_sat=15.0)
    sg_grey, _ = fb.texture_maps(fb.Plan(1, 90, 104), _dev(grey), **tp)
    assert np.max(np.abs(sg_grey.cpu().numpy() - orc.texture_maps(grey, **tp)[1])) <= 1e-4
    sg = sg_grey.repeat(3, 1, 1).contiguous()
    plan = fb.Plan(3, 90, 104)
    img = _dev(w.img)
    g1, g2 = torch.empty_like(img), torch.empty_like(img)
    out = fb.filter_texture_map(plan, img, sg, rho, N, second_scale=0.8, sharpen=sp, rho_sharpen=rs, pass1=g1, pass2=g2)
    torch.cuda.synchronize()
    sgh, g1, g2, out = sg.cpu().numpy(), g1.cpu().numpy(), g2.cpu().numpy(), out.cpu().numpy()
    sc = grey_scale(w.img)
    mx, nbad, _ = compare_guarded(g1, orc.fast(w.img, w.img, sgh, rho, N), sc)
    assert nbad == 0, f"pass 1: max |delta| = {mx} grey"
    mx, nbad, _ = compare_guarded(g2, orc.fast(g1, g1, (np.float32(0.8) * sgh).astype(np.float32), rho, N), sc)
    assert nbad == 0, f"pass 2: max |delta| = {mx} grey"
    th3, sg3 = fb.sharpen_maps(plan, _dev(g2), rs, **sp)
    torch.cuda.synchronize()
    mx, nbad, _ = compare_guarded(out, orc.fast(g2, th3.cpu().numpy(), sg3.cpu().numpy(), rs, N), sc)
    assert nbad == 0, f"pass 3: max |delta| = {mx} grey"
    ref = orc.texture_pipeline(w.img, rho, N, texture=dict(second_scale=0.8), sharpen=sp, rho_sharpen=rs, sigma=sgh)
    d = np.abs(out.astype(np.float64) - ref["out"]) / sc
    assert np.quantile(d, 0.999) <= TOL_GREY, f"end to end p99.9 = {np.quantile(d, 0.999)} grey, max {d.max()}"
    with pytest.raises(fb.FabfError):
        fb.filter_texture_map(plan, img, sg, rho, N, second_scale=0.0)


@pytest.mark.parametrize("kind,shape,rho,N", [
    ("voronoi", (1, 96, 130), 3, 5), ("texture", (2, 70, 81), 1, 8), ("rect", (1, 100, 100), 5, 2),
    ("float", (1, 80, 90), 3, 6), ("flat", (1, 40, 40), 2, 5), ("voronoi", (1, 130, 150), 10, 5),
    ("texture", (1, 140, 160), 12, 4), ("rect", (1, 60, 61), 2, 0), ("voronoi", (1, 64, 64), 0, 3)])
def test_gaussian_spatial_kernel(fb, orc, kind, shape, rho, N):
    """NEXT-1: Algorithm 1 with the Gaussian omega of eq.(4) on [-3 rho, 3 rho]^2
    (fabf_filter_gauss) against the oracle's weighted-histogram reference,
    every pixel; rho = 12 runs the 16 x 16 tile variant, rho = 0 the identity."""
    import torch

    w = workloads.random_case(*shape, seed=81 + rho, kind=kind, rho=rho, N=N)
    plan = fb.Plan(*w.shape)
    out = fb.filter_gauss(plan, _dev(w.img), _dev(w.theta), _dev(w.sigma), rho, N)
    torch.cuda.synchronize()
    o = orc.fast(w.img, w.theta, w.sigma, rho, N, spatial="gauss")
    mx, nbad, _ = compare_guarded(out.cpu().numpy(), o, grey_scale(w.img))
    assert nbad == 0, f"max |delta| = {mx} grey ({plan.last_fallback_count()} fallback pixels)"


def test_gaussian_spatial_kernel_fallback(fb, orc):
    """A flat area next to full contrast sends pixels to k_fallback_gauss (exact
    weighted moments); they match the oracle too."""
    import torch

    rng = np.random.default_rng(88)
    f = np.rint(rng.uniform(0, 255, (1, 90, 120)))
    f[:, :, :50] = np.rint(3 + rng.uniform(0, 2, (1, 90, 50)))
    f = f.astype(np.float32)
    th = (f + rng.uniform(-1, 1, f.shape)).astype(np.float32)
    sg = rng.uniform(0.5, 20, f.shape).astype(np.float32)
    plan = fb.Plan(*f.shape)
    out = fb.filter_gauss(plan, _dev(f), _dev(th), _dev(sg), 2, 10)
    torch.cuda.synchronize()
    assert plan.last_fallback_count() > 0
    o = orc.fast(f, th, sg, 2, 10, spatial="gauss")
    mx, nbad, _ = compare_guarded(out.cpu().numpy(), o, 1.0)
    assert nbad == 0, f"max |delta| = {mx} grey"


# ------------------------------------------------------------------ A/B switches of the library
_PLACEMENT_SCRIPT = r"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["FABF_ROOT"])
import paper_1811_02308_b200 as fb
import workloads
res = {}
for shape, rho in [((1, 150, 260), 7), ((2, 130, 300), 20), ((1, 200, 333), 30), ((1, 193, 517), 60)]:
    rng = np.random.default_rng(sum(shape) + rho)
    f = rng.normal(100, 60, shape).astype(np.float32)
    plan = fb.Plan(*shape)
    a, b = fb.bounds(plan, torch.from_numpy(f).cuda(), rho)
    res[f"f_{rho}"], res[f"a_{rho}"], res[f"b_{rho}"] = f, a.cpu().numpy(), b.cpu().numpy()
w = workloads.random_case(1, 160, 300, seed=5, kind="voronoi", rho=30, N=6)
plan = fb.Plan(*w.shape)
d = lambda x: torch.from_numpy(x).cuda()
res["g"] = fb.filter(plan, d(w.img), d(w.theta), d(w.sigma), w.rho, w.N).cpu().numpy()
np.savez(sys.argv[1], **res)
"""


@pytest.mark.parametrize("env", [{"FABF_BOUNDS": "tile"}, {"FABF_BOUNDS": "sep"}, {"FABF_PDL": "0"}])
def test_library_switches_bit_identical(fb, orc, tmp_path, env):
    """The library's A/B switches (read once at load: bounds by the 2-D tile
    kernel or the separable passes at every rho, programmatic dependent launch
    off) give the same bit-exact bounds (oracle scan) and the same filter
    output as the default placement."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for name, extra in (("default", {}), ("switched", env)):
        path = str(tmp_path / f"{name}.npz")
        e = dict(os.environ, FABF_ROOT=root, **extra)
        subprocess.run([sys.executable, "-c", _PLACEMENT_SCRIPT, path], env=e, check=True, timeout=600)
        outs[name] = np.load(path)
    for rho in (7, 20, 30, 60):
        f = outs["default"][f"f_{rho}"]
        ra, rb = orc.bounds(f, rho)
        for name in outs:
            assert np.array_equal(outs[name][f"a_{rho}"], ra), (name, rho)
            assert np.array_equal(outs[name][f"b_{rho}"], rb), (name, rho)
    assert np.array_equal(outs["default"]["g"], outs["switched"]["g"])
