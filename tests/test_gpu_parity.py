"""GPU parity: every stage of libhdrb200.so against the oracle / the
reference's golden fixtures, then the whole pair.

Bars (BASELINE.json north_star):
  * keypoints and match indices bit-exact; SSD scores <= 1e-12 relative;
  * RANSAC kept sets (and witness counts) identical under the same seed;
  * homographies within 1e-4 relative (observed ~1e-12);
  * f32 raster stages bit-exact; flow <= 1e-4 px; SSIM <= 1e-4;
  * warped / composite radiance <= 1e-3 max-abs.
"""

import numpy as np
import pytest
import torch

from golden_util import SCENES, digest, load, scene_inputs
from oracle import hdr_oracle as O
from harness import synth
from paper_1504_01441_b200 import densify, fusion, geometry, image, matcher, pipeline, weeding
from paper_1504_01441_b200.errors import RegistrationError

pytestmark = pytest.mark.gpu

FLOW_TOL = 1e-4
RADIANCE_TOL = 1e-3
SSIM_TOL = 1e-4
H_RTOL = 1e-4


@pytest.fixture(scope="module", params=SCENES)
def scene(request, cuda):
    fx = load(request.param)
    ref, src = scene_inputs(fx)
    return request.param, fx, ref, src


def rel_h(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max()


def assert_rows(got, want):
    """Match rows: coordinates bit-exact, score within 1e-12 relative."""
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    np.testing.assert_array_equal(got[:, :4], want[:, :4])
    np.testing.assert_allclose(got[:, 4], want[:, 4], rtol=1e-12, atol=1e-15)


def test_luminance_histogram_pyramid_bit_exact(scene):
    _, fx, ref, src = scene
    lum_ref = image.luminance(ref)
    assert digest(lum_ref) == str(fx["lum_ref_digest"])
    eq = image.match_histogram(image.luminance(src), lum_ref)
    assert digest(eq) == str(fx["eq_src_digest"])
    rp, sp = image.build_pyramid(lum_ref), image.build_pyramid(eq)
    assert [digest(a) for a in rp] + [digest(a) for a in sp] == list(fx["pyr_digests"])


def test_integral_bit_exact(scene):
    _, _, ref, _ = scene
    lum = O.luminance(ref)
    np.testing.assert_array_equal(image.integral(lum), O.integral(lum))


def test_cornerness_point_query(scene):
    """matcher.cornerness (matcher.py:50-61): KATs, random points vs the oracle,
    and the out-of-bounds ValueError."""
    img = np.zeros((32, 32), dtype=np.float32)
    img[:16, 16:] = 1.0
    img[16:, :16] = 1.0
    assert matcher.cornerness(image.integral(img), 16, 16) == (4.0, 1.0)
    edge = np.zeros((32, 32), dtype=np.float32)
    edge[:, 16:] = 1.0
    assert matcher.cornerness(image.integral(edge), 16, 16) == (2.0, 0.0)
    _, _, ref, _ = scene
    lum = O.luminance(ref)
    table = image.integral(lum)
    sat = O.integral(lum)
    h, w = lum.shape
    rng = np.random.default_rng(7)
    for half in (8, 3):
        for x, y in zip(rng.integers(half, w - half + 1, 20), rng.integers(half, h - half + 1, 20)):
            c, lo = O._quadrants(sat, np.array([x]), np.array([y]), half)
            assert matcher.cornerness(table, int(x), int(y), half) == (float(c[0]), float(lo[0]))
    for x, y in ((7, 20), (20, 7), (w - 7, 20), (20, h - 7)):
        with pytest.raises(ValueError, match="out of bounds"):
            matcher.cornerness(table, x, y)


def test_corners_matches_weeding_per_level(scene):
    _, fx, ref, src = scene
    lum_ref = O.luminance(ref)
    rp = O.pyramid(lum_ref)
    sp = O.pyramid(O.match_histogram(O.luminance(src), lum_ref))
    mp = matcher.MatcherParams()
    for lev in range(len(rp) - 1, -1, -1):
        h, w = rp[lev].shape
        corners = matcher.detect_corners(rp[lev], mp.tile, mp.threshold, mp.quadrant_half)
        np.testing.assert_array_equal(corners, fx[f"L{lev}_corners"])
        raw = matcher._match_level(rp[lev], sp[lev], fx[f"L{lev}_hpred"], mp)
        assert_rows(raw, fx[f"L{lev}_raw"])
        raw = fx[f"L{lev}_raw"]
        if len(raw) >= 4:
            res = weeding.weed_parallel(raw, (w, h), mp.weed_params(lev, w), 1)
            np.testing.assert_array_equal(res.kept, fx[f"L{lev}_kept"])
            np.testing.assert_array_equal(res.witness, fx[f"L{lev}_witness"])
        if f"L{lev}_hfit" in fx:
            hf = matcher.fit_matches_homography(raw[fx[f"L{lev}_kept"]], w, h)
            assert rel_h(hf, fx[f"L{lev}_hfit"]) < 1e-9


def test_corner_detector_both_sat_paths(cuda):
    """The tile-local detector runs only under the exactness certificate;
    tiny samples (real photos' dark pixels) break it and force numpy's
    sequential lattice SAT. Both must reproduce the oracle bit for bit."""
    st = synth.synth_stack(synth.working_spec(640, 480), 5)
    lum = O.luminance(st.ref)
    dark = lum.copy()
    rng = np.random.default_rng(0)
    idx = rng.integers(0, dark.size, 400)
    dark.ravel()[idx] = np.float32(1e-9) * rng.random(400, dtype=np.float32)
    for img in (lum, dark, (lum * np.float32(0.013)).astype(np.float32)):
        np.testing.assert_array_equal(matcher.detect_corners(img), O.detect_corners(img))


def test_fit_homography_and_inliers(cuda):
    rng = np.random.default_rng(3)
    for n in (4, 5, 9, 40, 300):
        p = rng.uniform(-1, 1, (n, 2))
        hm = np.array([[1.01, 0.02, 0.03], [-0.01, 0.99, -0.02], [0.01, -0.02, 1.0]])
        q = O._transfer  # noqa: F841 (oracle helper imported for symmetry)
        qh = np.c_[p, np.ones(n)] @ hm.T
        q = qh[:, :2] / qh[:, 2:]
        q += rng.normal(scale=1e-3, size=q.shape) if n > 4 else 0.0
        g = geometry.fit_homography(p, q)
        o = O.fit_homography(p, q)
        assert rel_h(g, o) < 1e-9, n
        np.testing.assert_array_equal(geometry.inlier_mask(g, p, q, 2e-3),
                                      O.inlier_mask(o, p, q, 2e-3))
    # degenerate: coincident, collinear-4 configurations
    from paper_1504_01441_b200.errors import DegenerateFit
    pts = np.array([[0.0, 0.0], [0.0, 0.0], [1.0, 1.0], [2.0, 0.5]])
    with pytest.raises(DegenerateFit):
        geometry.fit_homography(pts, pts)
    line = np.array([[0.0, 0.0], [1.0, 1.0], [2.0, 2.0], [3.0, 3.0]])
    with pytest.raises(O.DegenerateFit):
        O.fit_homography(line, line)
    with pytest.raises(DegenerateFit):
        geometry.fit_homography(line, line)


def test_homography_flow_bit_exact(cuda):
    hm = np.array([[1.001, 0.002, -0.01], [-0.003, 0.998, 0.004], [0.001, -0.002, 1.0]])
    np.testing.assert_array_equal(geometry.homography_pixel_flow(hm, 320, 240),
                                  O.homography_flow(hm, 320, 240))


def test_densify_warp_stages(scene):
    _, fx, ref, src = scene
    lum_ref = O.luminance(ref)
    h, w = lum_ref.shape
    m = fx["matches"]
    maps = densify.build_sparse_maps(m, w, h)
    omaps = O.sparse_maps(m, w, h)
    for a, b in zip((maps.pu, maps.pv, maps.n), omaps):
        np.testing.assert_array_equal(a, b)
    stacked = np.stack(omaps, axis=-1)
    sm = densify.dt_filter(lum_ref, stacked)
    osm = O.dt_filter(lum_ref, stacked)
    assert np.abs(sm - osm).max() < 1e-9
    hm = fx["homography"]
    flow = densify.densify_flow(lum_ref, maps, hm)
    oflow = O.densify_flow(lum_ref, omaps, hm)
    assert np.abs(flow - oflow).max() < FLOW_TOL
    # the warp itself is bit-exact given the same flow (f64 coordinates)
    warped, valid = densify.warp_image(src, oflow)
    owarped, ovalid = O.warp_image(src, oflow)
    np.testing.assert_array_equal(warped, owarped)
    np.testing.assert_array_equal(valid, ovalid)


@pytest.mark.parametrize("shape", [(480, 640), (37, 53), (37, 54), (1, 70), (70, 1), (2100, 33),
                                   (2100, 34), (1944, 130), (3000, 66), (4100, 6), (9000, 5)])
def test_dt_filter_all_column_paths(cuda, shape):
    """Every column-sweep implementation -- the register-resident cluster
    kernel with and without the cp.async band prefetch, and the chunk
    agg/link/apply path (very tall images) -- matches the
    oracle's sequential recursion for 1-3 planes, odd sizes and degenerate
    1-pixel axes."""
    from paper_1504_01441_b200 import _native
    h, w = shape
    rng = np.random.default_rng(h * 7 + w)
    guide = rng.random((h, w), dtype=np.float32)
    paths = [("dt_cluster_columns", 1, "dt_cols_prefetch", 1), ("dt_cluster_columns", 1, "dt_cols_prefetch", 0),
             ("dt_cluster_columns", 0, "dt_cols_prefetch", 1)]
    try:
        for k in (1, 2, 3):
            planes = rng.normal(size=(h, w, k))
            planes[rng.random((h, w)) < 0.9] = 0.0  # sparse like the splat maps
            want = O.dt_filter(guide, planes if k > 1 else planes[..., 0])
            for o1, v1, o2, v2 in paths:
                _native.check(_native.lib().hdr_set_option(o1.encode(), v1))
                _native.check(_native.lib().hdr_set_option(o2.encode(), v2))
                got = densify.dt_filter(guide, planes if k > 1 else planes[..., 0])
                assert np.abs(np.asarray(got) - want).max() < 1e-9, (k, o1, v1, o2, v2)
    finally:
        _native.lib().hdr_set_option(b"dt_cluster_columns", 1)
        _native.lib().hdr_set_option(b"dt_cols_prefetch", 1)


def test_sparse_first_row_pass_is_exact(cuda):
    """The CSR splat + first row pass built from it (the pair default) gives
    the same bits as the dense splat planes + the plain row pass, and as the
    sparse pass writing its sample-free rows instead of the first column
    sweep skipping them -- also when the context's planes still hold another
    pair's values (the skipped rows are never written by the row pass)."""
    from paper_1504_01441_b200 import _native
    st = synth.synth_stack(synth.working_spec(640, 480), 3)
    other = synth.synth_stack(synth.working_spec(640, 480), 5)
    pipeline.register_and_fuse(other.ref, other.src)  # leaves its planes behind
    a = pipeline.register_and_fuse(st.ref, st.src)
    try:
        _native.check(_native.lib().hdr_set_option(b"dt_sparse_first", 0))
        b = pipeline.register_and_fuse(st.ref, st.src)
        _native.check(_native.lib().hdr_set_option(b"dt_sparse_first", 1))
        _native.check(_native.lib().hdr_set_option(b"dt_skip_zero_rows", 0))
        c = pipeline.register_and_fuse(st.ref, st.src)
    finally:
        _native.lib().hdr_set_option(b"dt_sparse_first", 1)
        _native.lib().hdr_set_option(b"dt_skip_zero_rows", 1)
    for o in (b, c):
        np.testing.assert_array_equal(a.flow, o.flow)
        np.testing.assert_array_equal(a.composite, o.composite)


def test_ssim_and_fuse_stages(scene):
    _, fx, ref, src = scene
    o = O.register_and_fuse(ref, src)
    lum_ref = O.luminance(ref)
    s = pipeline.make_ssim(lum_ref, o.warped, pipeline.PipelineParams())
    assert np.abs(s - o.ssim).max() < SSIM_TOL
    q = fusion.quality_weights(ref)
    oq = O.quality_weights(ref)
    assert np.abs(q - oq).max() / oq.max() < 1e-5
    comp = fusion.fuse(ref, o.warped, o.ssim, o.valid.astype(np.float32))
    assert np.abs(comp - o.composite).max() < RADIANCE_TOL


def check_pair(res, o):
    """The whole pair: sparse results exact, dense outputs through
    test_gpu_headline.check_dense (valid identical; SSIM 1e-4 outside the
    window of a quantisation flip of the warped luminance)."""
    from test_gpu_headline import check_dense
    assert res.level_counts == o.level_counts
    assert_rows(res.raw_matches, o.raw_matches)
    assert_rows(res.matches, o.matches)
    assert (res.homography is None) == (o.homography is None)
    if o.homography is not None:
        assert rel_h(res.homography, o.homography) < H_RTOL
    assert res.flow.dtype == np.float32 and res.ssim.dtype == np.float64
    assert res.valid.dtype == bool and res.composite.dtype == np.float32
    check_dense(res, o)


def test_register_and_fuse_end_to_end(scene):
    _, fx, ref, src = scene
    res = pipeline.register_and_fuse(ref, src)
    o = O.register_and_fuse(ref, src)
    check_pair(res, o)
    np.testing.assert_array_equal(np.asarray(res.level_counts), fx["level_counts"])


def test_graph_replay_matches_eager(cuda):
    st = synth.synth_stack(synth.working_spec(640, 480), 0)
    ref = torch.from_numpy(st.ref).cuda()
    src = torch.from_numpy(st.src).cuda()
    p = pipeline.PipelineParams()
    a = pipeline.PairBuffers(640, 480, 0)
    b = pipeline.PairBuffers(640, 480, 0)
    pipeline.enqueue_pair(ref, src, p, a, graph=False)
    for _ in range(2):
        pipeline.enqueue_pair(ref, src, p, b, graph=True)
    torch.cuda.synchronize()
    for name in ("composite", "flow", "warped", "valid", "ssim", "info"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name


def test_graph_cache_survives_parameter_changes(cuda):
    """A cached pair graph replays against the key / fit / tap buffers it was
    captured with: calls with more RANSAC iterations, another seed or another
    SSIM window in between (which allocate new parameter sets) must not
    change what the first graph computes."""
    st = synth.synth_stack(synth.working_spec(640, 480), 0)
    ref = torch.from_numpy(st.ref).cuda()
    src = torch.from_numpy(st.src).cuda()
    p = pipeline.PipelineParams()
    a = pipeline.PairBuffers(640, 480, 0)
    b = pipeline.PairBuffers(640, 480, 0)
    pipeline.enqueue_pair(ref, src, p, a, graph=True)
    torch.cuda.synchronize()
    first = {n: getattr(a, n).clone() for n in ("composite", "flow", "ssim", "matches", "info")}
    for q in (pipeline.PipelineParams(iterations=512, coarse_iterations=128),
              pipeline.PipelineParams(seed=7), pipeline.PipelineParams(ssim_window=7, ssim_sigma=1.0)):
        pipeline.enqueue_pair(ref, src, q, b, graph=True)
    pipeline.enqueue_pair(ref, src, p, a, graph=True)
    torch.cuda.synchronize()
    for n, t in first.items():
        assert torch.equal(getattr(a, n), t), n


def test_concurrent_threads_are_independent(cuda):
    """The drop-in is re-entrant like the reference's pure functions: two
    host threads calling register_and_fuse at once on different scenes get
    exactly what each gets alone (each thread owns its workspace)."""
    import threading
    scenes = [synth.synth_stack(synth.working_spec(640, 480), s) for s in (0, 3)]
    alone = [pipeline.register_and_fuse(st.ref, st.src) for st in scenes]
    got = [[None] * 3 for _ in scenes]
    errs = []

    def work(i):
        try:
            for r in range(3):
                got[i][r] = pipeline.register_and_fuse(scenes[i].ref, scenes[i].src)
        except Exception as exc:  # pragma: no cover - surfaced below
            errs.append(exc)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i in range(2):
        for r in range(3):
            for n in ("composite", "flow", "ssim", "matches", "valid"):
                np.testing.assert_array_equal(getattr(got[i][r], n), getattr(alone[i], n))


def test_async_enqueues_on_two_streams(cuda):
    """enqueue_pair on two streams without a host sync in between: the shared
    thread context orders the second after the first (event), so both pairs
    come out right."""
    scenes = [synth.synth_stack(synth.working_spec(640, 480), s) for s in (0, 3)]
    alone = [pipeline.register_and_fuse(st.ref, st.src) for st in scenes]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    bufs = [pipeline.PairBuffers(640, 480, 0) for _ in scenes]
    ins = [(torch.from_numpy(st.ref).cuda(), torch.from_numpy(st.src).cuda()) for st in scenes]
    torch.cuda.synchronize()
    for k, s in enumerate((s1, s2)):
        pipeline.enqueue_pair(ins[k][0], ins[k][1], pipeline.PipelineParams(), bufs[k], stream=s)
    torch.cuda.synchronize()
    for k in range(2):
        np.testing.assert_array_equal(bufs[k].composite.cpu().numpy(), alone[k].composite)


def test_registration_error_parity(cuda):
    st = synth.synth_stack(synth.SceneSpec(), 0)
    with pytest.raises(RegistrationError, match="only 0 reliable matches at full resolution"):
        pipeline.register_and_fuse(st.ref, st.src)


def test_config_and_shape_errors(cuda):
    from paper_1504_01441_b200.errors import ConfigError
    a = np.zeros((200, 200, 3), np.float32)
    with pytest.raises(ConfigError):
        pipeline.register_and_fuse(a, a, pipeline.PipelineParams(tile=8))
    with pytest.raises(ConfigError):
        pipeline.register_and_fuse(a, np.zeros((200, 201, 3), np.float32))
    with pytest.raises(ValueError):
        pipeline.register_and_fuse(np.zeros((90, 200, 3), np.float32),
                                   np.zeros((90, 200, 3), np.float32))


def test_gray_inputs_and_torch_inputs(cuda):
    st = synth.synth_stack(synth.working_spec(320, 240), 2)
    g_ref, g_src = st.ref.mean(axis=2).astype(np.float32), st.src.mean(axis=2).astype(np.float32)
    o = None
    try:
        o = O.register_and_fuse(g_ref, g_src)
    except O.RegistrationError:
        with pytest.raises(RegistrationError):
            pipeline.register_and_fuse(g_ref, g_src)
    if o is not None:
        check_pair(pipeline.register_and_fuse(g_ref, g_src), o)
    t = pipeline.register_and_fuse(torch.from_numpy(st.ref).cuda(), torch.from_numpy(st.src).cuda())
    assert isinstance(t.composite, torch.Tensor) and t.composite.is_cuda
    n = pipeline.register_and_fuse(st.ref, st.src)
    np.testing.assert_array_equal(t.composite.cpu().numpy(), n.composite)


def test_batch_runner_raw_path(cuda):
    """run_host_raw (raw 8-bit samples in, save_png's 8-bit composite out)
    equals decode -> register_and_fuse -> quantise pair for pair."""
    from paper_1504_01441_b200.runner import BatchRunner
    from paper_1504_01441_b200 import _native, fileio
    w, h = 320, 240
    q8 = lambda a: np.clip(np.floor(a.astype(np.float64) * 255.0 + 0.5), 0, 255).astype(np.uint8)
    stacks = [synth.synth_stack(synth.working_spec(w, h), s) for s in (2, 7)]
    raws = [(q8(st.ref), q8(st.src)) for st in stacks]
    want = []
    for a, b in raws:
        fa = (a.astype(np.float64) / 255.0).astype(np.float32)
        fb = (b.astype(np.float64) / 255.0).astype(np.float32)
        want.append(fileio.quantize_u8(pipeline.register_and_fuse(fa, fb).composite).cpu().numpy())
    r = BatchRunner(w, h, streams=2)
    n = 5
    hp = [(torch.from_numpy(raws[k % 2][0]).pin_memory(), torch.from_numpy(raws[k % 2][1]).pin_memory())
          for k in range(n)]
    ho = [(torch.empty((h, w, 3), dtype=torch.uint8).pin_memory(),
           torch.empty((_native.INFO_WORDS,), dtype=torch.int32).pin_memory()) for _ in range(n)]
    for _ in range(2):
        r.run_host_raw(hp, ho, 8)
    torch.cuda.synchronize()
    for k in range(n):
        assert int(ho[k][1][0]) == 0
        np.testing.assert_array_equal(ho[k][0].numpy(), want[k % 2])
    r.close()


def test_batch_runner_host_and_device_paths(cuda):
    """The throughput runner (several streams, graph replays, double-buffered
    host path) returns, pair for pair, what the single-pair API returns."""
    from paper_1504_01441_b200.runner import BatchRunner
    from paper_1504_01441_b200.pipeline import PairBuffers
    from paper_1504_01441_b200 import _native
    w, h = 320, 240
    stacks = [synth.synth_stack(synth.working_spec(w, h), s) for s in (2, 7, 9)]
    want = [pipeline.register_and_fuse(st.ref, st.src) for st in stacks]
    r = BatchRunner(w, h, streams=2)
    n = 7  # odd, > 2 slots per stream: exercises slot reuse ordering
    hp = [(torch.from_numpy(stacks[k % 3].ref).pin_memory(),
           torch.from_numpy(stacks[k % 3].src).pin_memory()) for k in range(n)]
    ho = [(torch.empty((h, w, 3), dtype=torch.float32).pin_memory(),
           torch.empty((_native.INFO_WORDS,), dtype=torch.int32).pin_memory()) for _ in range(n)]
    for _ in range(2):
        r.run_host(hp, ho)
    torch.cuda.synchronize()
    for k in range(n):
        np.testing.assert_array_equal(ho[k][0].numpy(), np.asarray(want[k % 3].composite))
    dev = [(a.cuda(), b.cuda()) for a, b in hp]
    outs = [PairBuffers(w, h, torch.cuda.current_device()) for _ in range(n)]
    r.run_device(dev, outs)
    torch.cuda.synchronize()
    for k in range(n):
        np.testing.assert_array_equal(outs[k].composite.cpu().numpy(),
                                      np.asarray(want[k % 3].composite))
    r.close()
