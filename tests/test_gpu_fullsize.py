"""Full-size parity at BASELINE.json's own shapes, in the launch configuration
bench.py times, every compared pixel against the oracle.

* config 4 (3840x2160, rho=20, N=8): every one of the 8,294,400 pixels;
* config 5 (32 x 1024^2): the fallback-heaviest (rho, N) cells, the whole batch
  filtered in one call, four frames (0, 11, 22, 31) compared pixel by pixel;
* regressions at band / segment starts (row 64k - rho - 1 outside every window
  of the segment) through fabf_filter and fabf_filter_host, and the fallback
  count of fabf_filter_host summed over its bands.

The oracle sums eq.(22) over the window's histogram (oracle/fabf_oracle.c), which
is what makes whole frames affordable here.
"""
import numpy as np
import pytest

import workloads
from parity import compare_guarded

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


def _filter(fb, w, flags=0):
    import torch

    plan = fb.Plan(*w.shape, flags)
    out = fb.filter(plan, _dev(w.img), _dev(w.theta), _dev(w.sigma), w.rho, w.N)
    torch.cuda.synchronize()
    return out.cpu().numpy(), plan


@pytest.fixture(scope="module")
def cfg4(orc):
    w = workloads.config(4)
    return w, orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)


@pytest.mark.parametrize("fused", [False, True])
def test_config4_every_pixel(fb, cfg4, fused):
    """Both bounds placements: k_bounds + k_filter (the default at rho = 20)
    and FABF_FLAG_FUSED (bounds inside k_filter, one pass over f, theta, sigma)."""
    w, o = cfg4
    out, plan = _filter(fb, w, fb.FLAG_FUSED if fused else 0)
    mx, nbad, err = compare_guarded(out, o, 1.0)
    assert nbad == 0, f"max |delta| = {mx} grey"
    assert np.isfinite(out).all()
    ident = (o["code"] & 1) > 0
    assert np.array_equal(out[ident], w.img[ident])
    print(f"config 4 every pixel (fused={fused}): max |delta| {mx:.3e} grey, "
          f"p99.9 {np.quantile(err, 0.999):.3e}, fallback pixels {plan.last_fallback_count()}, "
          f"kernels {plan.last_launch_count()}")


FRAMES = (0, 11, 22, 31)


@pytest.mark.parametrize("gen,rho,N,expect_fallback,fused", [
    ("texture", 40, 8, True, False), ("texture", 40, 10, True, False), ("texture", 20, 10, True, False),
    ("rectangles", 2, 10, True, False), ("texture", 40, 10, True, True)])
def test_config5_cells_full_batch(fb, orc, gen, rho, N, expect_fallback, fused):
    w = workloads.config5(rho, N, batch=32, size=1024, generator=gen)
    out, plan = _filter(fb, w, fb.FLAG_FUSED if fused else 0)
    nfb = plan.last_fallback_count()
    if expect_fallback:
        assert nfb > 0, "expected pixels on the exact-moment fallback"
    sub = np.array(FRAMES)
    o = orc.fast(w.img[sub], w.theta[sub], w.sigma[sub], w.rho, w.N)
    mx, nbad, _ = compare_guarded(out[sub], o, 1.0)
    assert nbad == 0, f"{gen} rho={rho} N={N}: max |delta| = {mx} grey ({nfb} fallback pixels)"
    assert np.isfinite(out).all()
    print(f"config 5 {gen} rho={rho} N={N} fused={fused}: max |delta| {mx:.3e} grey over frames {FRAMES}, "
          f"{nfb} fallback pixels in the batch")


def _outlier_rows_image(H, W, rho, seed):
    """Flat, low-noise image (levels 128..133) with full-contrast outlier rows at
    y = 64k - rho - 1: those rows lie outside every window of a segment that
    starts at row 64k, and far outside its centring range."""
    rng = np.random.default_rng(seed)
    f = np.rint(128 + rng.uniform(0, 5, (H, W)))
    for y in range(64 - rho - 1, H, 64):
        f[y] = np.where(np.arange(W) % 2 == 0, 0.0, 255.0)
    th = f + rng.uniform(-2, 2, f.shape)
    sg = rng.uniform(3, 30, f.shape)
    return [a.astype(np.float32)[None] for a in (f, th, sg)]


@pytest.mark.parametrize("rho,N,fused", [(20, 8, False), (9, 10, False), (4, 8, False), (20, 8, True)])
def test_segment_start_outlier_rows(fb, orc, rho, N, fused):
    f, th, sg = _outlier_rows_image(64 * 9 + 17, 300, rho, 900 + rho)
    w = workloads.Workload("outlier_rows", f, th, sg, rho, N)
    out, _ = _filter(fb, w, fb.FLAG_FUSED if fused else 0)
    o = orc.fast(f, th, sg, rho, N)
    mx, nbad, _ = compare_guarded(out, o, 1.0)
    assert nbad == 0, f"fabf_filter: max |delta| = {mx} grey"
    plan = fb.Plan(*f.shape)
    host_out = np.empty_like(f)
    fb.filter_host(plan, f, th, sg, rho, N, host_out)  # bands start at multiples of 64 rows
    mx, nbad, _ = compare_guarded(host_out, o, 1.0)
    assert nbad == 0, f"fabf_filter_host: max |delta| = {mx} grey"


def test_host_fallback_count_sums_bands(fb, orc):
    """fabf_last_fallback_count after fabf_filter_host counts every band of every
    image (it equals the device entry point's count on the same input)."""
    rng = np.random.default_rng(31)
    B, H, W = 2, 64 * 7, 256
    f = np.rint(rng.uniform(0, 255, (B, H, W)))
    f[:, :, :100] = np.rint(3 + rng.uniform(0, 2, (B, H, 100)))  # flat next to full contrast
    # every row holds 0 and 255 in the first strip: every segment of it has the
    # same centring range, so the fallback flags do not depend on where the
    # device (work chunks) or host (row bands) path starts its segments
    f[:, :, 100], f[:, :, 101] = 0.0, 255.0
    f = f.astype(np.float32)
    th = (f + rng.uniform(-1, 1, f.shape)).astype(np.float32)
    sg = rng.uniform(0.5, 20, f.shape).astype(np.float32)
    w = workloads.Workload("fallback_bands", f, th, sg, 2, 10)
    out, plan = _filter(fb, w)
    n_dev = plan.last_fallback_count()
    assert n_dev > 0
    host_out = np.empty_like(f)
    fb.filter_host(plan, f, th, sg, 2, 10, host_out)
    assert plan.last_fallback_count() == n_dev
    o = orc.fast(f, th, sg, 2, 10)
    mx, nbad, _ = compare_guarded(host_out, o, 1.0)
    assert nbad == 0, f"max |delta| = {mx} grey"


def test_binding_refuses_wrong_dtype_and_size(fb):
    plan = fb.Plan(1, 32, 32)
    good = np.zeros((1, 32, 32), np.float32)
    out = np.empty_like(good)
    with pytest.raises(fb.FabfError):
        fb.filter_host(plan, good.astype(np.int32), good, good, 2, 3, out)
    with pytest.raises(fb.FabfError):
        fb.filter_host(plan, np.zeros((1, 16, 32), np.float32), good, good, 2, 3, out)
    with pytest.raises(fb.FabfError):
        fb.filter(plan, _dev(np.zeros((1, 16, 32))), _dev(good), _dev(good), 2, 3)
