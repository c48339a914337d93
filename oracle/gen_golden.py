"""Generate tests/golden/*.npz by running the REAL reference (`hdrflow`).

TEST INFRASTRUCTURE ONLY. Runs in the build container, where the reference
is importable from /root/reference/pkg/src; the fixtures it writes are what
pins the oracle (tests/test_oracle_golden.py) on any host.

The reference needs one shim to return from a successful registration:
`pipeline.fit_fallback` uses `fit_matches_homography`, which pipeline.py
never imports (pipeline.py:148 vs :18-24).

usage: python oracle/gen_golden.py [--ref /root/reference/pkg/src]
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from harness import synth  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
STRIDE = 8  # dense outputs: full-array digests + a 1-in-8 lattice sample


def sub(a, stride=STRIDE):
    s = np.ascontiguousarray(a[::stride, ::stride])
    return s.astype(np.float32) if s.dtype == np.float64 else s

# (name, width, height, rotation_deg, seed)
SCENES = [
    ("vga_s0", 640, 480, 0.0, 0),
    ("vga_rot_s1", 640, 480, 0.5, 1),
    ("qvga_s2", 320, 240, 0.0, 2),
    ("r960_s3", 960, 720, 0.25, 3),
]

# BASELINE.json's headline shapes, pinned to the
# real reference: dense outputs keep full-array digests, per-level traces
# and a 1-in-32 lattice sample (fixtures stay small)
BIG_SCENES = [
    ("c2_5mp_s0", 2592, 1944, 0.0, 0),
    ("c4_12mp_s0", 4000, 3000, 0.0, 0),
]
BIG_STRIDE = 32


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()


def load_reference(path):
    sys.path.insert(0, path)
    from hdrflow import image, matcher, pipeline  # noqa: F401
    pipeline.fit_matches_homography = matcher.fit_matches_homography
    import hdrflow
    return hdrflow


def scene_fixture(hf, w, h, rot, seed, stride=STRIDE):
    from hdrflow import densify, fusion, image, matcher, pipeline, weeding
    st = synth.synth_stack(synth.working_spec(w, h, rotation_deg=rot), seed)
    ref, src = st.ref, st.src
    params = pipeline.PipelineParams()
    out = {"inputs_digest": np.array([digest(ref), digest(src)])}
    lum_ref = image.luminance(ref)
    lum_src = image.luminance(src)
    eq = image.match_histogram(lum_src, lum_ref)
    rp = image.build_pyramid(lum_ref, params.max_levels)
    sp = image.build_pyramid(eq, params.max_levels)
    out["lum_ref_digest"] = np.array(digest(lum_ref))
    out["eq_src_digest"] = np.array(digest(eq))
    out["pyr_digests"] = np.array([digest(a) for a in rp] + [digest(a) for a in sp])
    out["n_levels"] = np.array(len(rp))
    # per-level trace, re-running the reference's own stages
    mp = params.matcher_params()
    h_pred = np.eye(3)
    for lev in range(len(rp) - 1, -1, -1):
        lr, ls = rp[lev], sp[lev]
        hh, ww = lr.shape
        out[f"L{lev}_corners"] = matcher.detect_corners(lr, mp.tile, mp.threshold, mp.quadrant_half)
        out[f"L{lev}_hpred"] = h_pred.copy()
        raw = matcher._match_level(lr, ls, h_pred, mp)
        out[f"L{lev}_raw"] = raw
        kept = np.zeros(0, dtype=np.int64)
        if len(raw) >= 4:
            res = weeding.weed_parallel(raw, (ww, hh), mp.weed_params(lev, ww), mp.workers)
            kept, wit = res.kept, res.witness
            out[f"L{lev}_witness"] = wit
        out[f"L{lev}_kept"] = kept
        weeded = raw[kept] if len(raw) >= 4 else np.zeros((0, 5))
        if len(weeded) >= 4:
            try:
                h_pred = matcher.fit_matches_homography(weeded, ww, hh)
                out[f"L{lev}_hfit"] = h_pred
            except Exception:
                pass
    r = pipeline.register_and_fuse(ref, src, params)
    for k in ("matches", "raw_matches"):
        out[k] = getattr(r, k)
    out["homography"] = r.homography if r.homography is not None else np.zeros((0, 3))
    out["level_counts"] = np.array(r.level_counts, dtype=np.int64)
    for k in ("composite", "flow", "warped", "valid", "ssim"):
        a = getattr(r, k)
        out[f"{k}_digest"] = np.array(digest(a))
        out[f"{k}_sub"] = sub(a, stride)
    # staged intermediates on the reference's own path
    maps = densify.build_sparse_maps(r.matches, w, h)
    sm = densify.dt_filter(lum_ref, np.stack([maps.pu, maps.pv, maps.n], axis=-1),
                           params.sigma_s, params.sigma_r, params.passes)
    out["smooth_digest"] = np.array(digest(sm))
    out["smooth_sub"] = sub(sm, stride)
    wr, ws = fusion.fusion_weights(ref, r.warped, r.ssim, r.valid.astype(np.float32))
    out["wref_sub"] = sub(wr, stride)
    out["wsrc_sub"] = sub(ws, stride)
    # the Ntilde-floor regime (densify.py:131-139): pixels falling back to the
    # global-H flow, and how many sit within 1e-3 relative of the floor
    nt = sm[..., 2]
    out["floor_fallback"] = np.array(int((nt <= params.normalization_floor).sum()))
    out["floor_near"] = np.array(int((np.abs(nt - params.normalization_floor)
                                      <= 1e-3 * params.normalization_floor).sum()))
    out["stride"] = np.array(stride)
    return out


# file-path cases (pipeline.run_hdr): (name, mode, exposures, swap inputs)
FILE_CASES = [
    ("file_rgb8", "RGB", (1.0, 4.0), False),
    ("file_rgb8_tie", "RGB", (2.0, 2.0), True),
    ("file_gray16", "I;16", (4.0, 1.0), True),
]


def write_scene_pngs(directory, mode, swap, w=640, h=480, seed=5):
    """The C1 scene written as PNG files the way a camera pipeline would
    store it (8-bit RGB or 16-bit grey); deterministic, so tests regenerate
    the same files instead of committing them."""
    from PIL import Image
    st = synth.synth_stack(synth.working_spec(w, h), seed)
    frames = [st.ref, st.src]
    if swap:
        frames = frames[::-1]
    paths = []
    for i, f in enumerate(frames):
        path = os.path.join(directory, f"in{i}.png")
        if mode == "RGB":
            data = np.clip(np.floor(f.astype(np.float64) * 255.0 + 0.5), 0, 255).astype(np.uint8)
            Image.fromarray(data, mode="RGB").save(path, format="PNG")
        else:
            lum = (0.299 * f[..., 0] + 0.587 * f[..., 1] + 0.114 * f[..., 2]).astype(np.float64)
            data = np.clip(np.floor(lum * 65535.0 + 0.5), 0, 65535).astype(np.uint16)
            Image.fromarray(data, mode="I;16").save(path, format="PNG")
        paths.append(path)
    return paths


def file_fixture(name, mode, exposures, swap):
    import tempfile
    from PIL import Image
    from hdrflow import fileio, pipeline
    with tempfile.TemporaryDirectory() as d:
        paths = write_scene_pngs(d, mode, swap)
        outp = os.path.join(d, "out.png")
        cfg = pipeline.PipelineConfig(inputs=paths, exposures=list(exposures), output=outp)
        r = pipeline.run_hdr(cfg)
        with Image.open(outp) as im:
            comp8 = np.asarray(im)
        imgs = [fileio.load_png(p) for p in paths]
        return {"inputs_digest": np.array([digest(a) for a in imgs]),
                "composite_u8_digest": np.array(digest(comp8)),
                "composite_u8_sub": comp8[::STRIDE, ::STRIDE].copy(),
                "composite_digest": np.array(digest(r.composite)),
                "level_counts": np.array(r.level_counts, dtype=np.int64),
                "exposures": np.array(exposures), "swap": np.array(swap),
                "mode": np.array(mode)}


def format_fixture():
    """Bytes written by the reference's PFM / match-CSV writers for small
    seeded arrays (pins paper_1504_01441_b200.fileio's writers)."""
    import tempfile
    from hdrflow import fileio
    rng = np.random.default_rng(11)
    grey = rng.random((5, 7), dtype=np.float32)
    colour = rng.random((4, 3, 3), dtype=np.float32)
    matches = np.concatenate([rng.random((6, 4)) * 640, rng.random((6, 1))], axis=1)
    out = {"grey": grey, "colour": colour, "matches": matches}
    with tempfile.TemporaryDirectory() as d:
        for name, fn, arr in (("grey", fileio.save_pfm, grey), ("colour", fileio.save_pfm, colour),
                              ("matches", fileio.save_matches_csv, matches)):
            path = os.path.join(d, name)
            fn(path, arr)
            out[f"{name}_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    return out


def stack_frames(w, h, seed):
    """BASELINE config C3 at any size: the -2 / 0 / +2 EV stack of SURVEY.md
    §8(d) -- the base frame and its +2 and +4 stop renderings (one seed, so
    the base frame is shared), in the order (+2, base, +4)."""
    a = synth.synth_stack(synth.working_spec(w, h, stops=2.0), seed)
    b = synth.synth_stack(synth.working_spec(w, h, stops=4.0), seed)
    assert np.array_equal(a.ref, b.ref)
    return [a.src, a.ref, b.src], [4.0, 1.0, 16.0]


def stack_fixture(w, h, seed, stride=STRIDE):
    """k-way stack composed from the REAL reference's functions: metering's
    reference choice, a pairwise register_and_fuse per source (for its
    warped frame, SSIM and validity), quality_weights, the pyramids and
    collapse_pyramid (the composition the oracle's fuse_stack restates)."""
    from hdrflow import fusion, metering, pipeline
    frames, exposures = stack_frames(w, h, seed)
    k = metering.choose_reference(frames, exposures)
    ref = frames[k]
    warped, ssims, valids, counts = [ref], [], [], []
    for f, src in enumerate(frames):
        if f == k:
            continue
        r = pipeline.register_and_fuse(ref, src)
        warped.append(r.warped)
        ssims.append(r.ssim)
        valids.append(r.valid.astype(np.float32))
        counts.append(np.array(r.level_counts, dtype=np.int64))
    levels = fusion.default_fusion_levels(h, w)
    ws = [fusion.quality_weights(ref)]
    for f in range(1, len(warped)):
        ws.append(fusion.quality_weights(warped[f]) * np.clip(ssims[f - 1], 0.0, 1.0)
                  * np.asarray(valids[f - 1], dtype=np.float64))
    tot = ws[0]
    for x in ws[1:]:
        tot = tot + x
    ws = [x / tot for x in ws]
    laps = [fusion.laplacian_pyramid(x, levels) for x in warped]
    gps = [fusion.gaussian_pyramid(x, levels) for x in ws]
    blended = []
    for lev in range(len(laps[0])):
        acc = gps[0][lev][:, :, None] * laps[0][lev]
        for f in range(1, len(warped)):
            acc = acc + gps[f][lev][:, :, None] * laps[f][lev]
        blended.append(acc)
    comp = np.clip(fusion.collapse_pyramid(blended), 0.0, 1.0).astype(np.float32)
    out = {"scene": np.array([w, h, seed]), "reference_index": np.array(k),
           "composite_digest": np.array(digest(comp)), "composite_sub": sub(comp, stride),
           "stride": np.array(stride)}
    for i, c in enumerate(counts):
        out[f"level_counts_{i}"] = c
    return out


def metering_images():
    """Seeded frames spanning the three select_offset outcomes, RGB and grey."""
    rng = np.random.default_rng(21)
    out = []
    for scale in (1.0, 0.25, 0.08, 0.02):
        img = (rng.random((60, 80, 3)) * scale).astype(np.float32)
        out.append(img)
        out.append(np.ascontiguousarray(img[..., 1]))
    return out


def metering_fixture():
    from hdrflow import metering
    imgs = metering_images()
    offs = [metering.select_offset(x) for x in imgs]
    plans = [metering.plan_stack([imgs[i], imgs[i + 2]], [1.0, 1.0]) for i in range(0, 6, 2)]
    return {"offsets": np.array(offs),
            "plans": np.array([[p.offset_stops, p.reference_index] for p in plans])}


# rows wider than the shared-memory row kernels (the pair pipeline's
# sequential row twin, k_twins.cu) -- pinned like the headline shapes
WIDE_SCENES = [("wide_7200x1000_s0", 7200, 1000, 0.0, 0)]


def twins_fixture():
    """Stage twins with the general arguments the reference accepts and the
    pair pipeline never passes: multi-channel / float64 guides and any plane
    count for dt_filter, any channel count for warp_image, batched rect_sum,
    quantize_256 and downsample on float32/float64, apply_homography and
    symmetric_transfer_error (image.py:47-93, geometry.py:80-115,
    densify.py:59-174)."""
    from hdrflow import densify, geometry, image
    r = np.random.default_rng(11)
    fx = {}
    g3 = r.random((37, 53, 3)).astype(np.float32)
    d4 = r.random((37, 53, 4))
    fx["dt_g3_guide"], fx["dt_g3_data"] = g3, d4
    fx["dt_g3_out"] = densify.dt_filter(g3, d4, 40.0, 0.3, 2)
    g64 = r.random((29, 31))
    d1 = r.random((29, 31))
    fx["dt_g64_guide"], fx["dt_g64_data"] = g64, d1
    fx["dt_g64_out"] = densify.dt_filter(g64, d1)
    g9 = r.random((20, 24, 9)).astype(np.float32)
    d2 = r.random((20, 24, 2))
    fx["dt_g9_guide"], fx["dt_g9_data"] = g9, d2
    fx["dt_g9_out"] = densify.dt_filter(g9, d2, 25.0, 0.1, 3)
    g1 = r.random((23, 41)).astype(np.float32)
    d5 = r.random((23, 41, 5))
    fx["dt_k5_guide"], fx["dt_k5_data"] = g1, d5
    fx["dt_k5_out"] = densify.dt_filter(g1, d5, 60.0, 0.2, 3)
    for c in (2, 4, 5):
        src = r.random((30, 40, c)).astype(np.float32)
        flow = (r.random((30, 40, 2)) * 8 - 4).astype(np.float32)
        warped, valid = densify.warp_image(src, flow)
        fx[f"warp{c}_src"], fx[f"warp{c}_flow"] = src, flow
        fx[f"warp{c}_out"], fx[f"warp{c}_valid"] = warped, valid
    img = r.random((17, 23)).astype(np.float32)
    t = image.integral(img)
    q = np.sort(r.integers(0, 18, (2, 50)), axis=0), np.sort(r.integers(0, 24, (2, 50)), axis=0)
    fx["rs_table"] = t
    fx["rs_q"] = np.stack([q[1][0], q[0][0], q[1][1], q[0][1]])
    fx["rs_out"] = image.rect_sum(t, q[1][0], q[0][0], q[1][1], q[0][1])
    fx["rs_scalar"] = np.float64(image.rect_sum(t, 3, 2, 19, 11))
    x32 = np.concatenate([r.random(200).astype(np.float32) * 1.4 - 0.2,
                          (np.arange(256, dtype=np.float32) + 0.5) / 255,
                          np.array([0.0, 1.0, -0.0, 2.0], np.float32)])
    x64 = np.concatenate([r.random(200) * 1.4 - 0.2, (np.arange(256) + 0.5) / 255])
    fx["q32_in"], fx["q32_out"] = x32, image.quantize_256(x32)
    fx["q64_in"], fx["q64_out"] = x64, image.quantize_256(x64)
    ds3 = r.random((21, 17, 3)).astype(np.float32)
    ds64 = r.random((14, 19, 2))
    fx["ds3_in"], fx["ds3_out"] = ds3, image.downsample(ds3)
    fx["ds64_in"], fx["ds64_out"] = ds64, image.downsample(ds64)
    hm = np.eye(3) + r.normal(size=(3, 3)) * 0.05
    pts = r.random((4, 25, 2)) * 100
    fx["h"], fx["h_pts"], fx["h_out"] = hm, pts, geometry.apply_homography(hm, pts)
    rp, sp = r.random((60, 2)) * 100, r.random((60, 2)) * 100
    fx["ste_ref"], fx["ste_src"] = rp, sp
    fx["ste_out"] = geometry.symmetric_transfer_error(hm, rp, sp)
    return fx


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--wide", action="store_true",
                    help="only the wide-row scene (7200x1000) and the stage-twin fixture")
    ap.add_argument("--big", action="store_true",
                    help="only the headline-size fixtures (C2 5MP, C4 12MP, C3 5MP stack; minutes of CPU)")
    args = ap.parse_args()
    hf = load_reference(args.ref)
    os.makedirs(GOLDEN, exist_ok=True)
    if args.wide:
        np.savez_compressed(os.path.join(GOLDEN, "twins.npz"), **twins_fixture())
        print("twins done")
        for name, w, h, rot, seed in WIDE_SCENES:
            fx = scene_fixture(hf, w, h, rot, seed, BIG_STRIDE)
            fx["scene"] = np.array([w, h, rot, seed], dtype=np.float64)
            np.savez_compressed(os.path.join(GOLDEN, f"{name}.npz"), **fx)
            print(name, fx["level_counts"].tolist(), int(fx["floor_fallback"]), int(fx["floor_near"]))
        return
    if args.big:
        for name, w, h, rot, seed in BIG_SCENES:
            fx = scene_fixture(hf, w, h, rot, seed, BIG_STRIDE)
            fx["scene"] = np.array([w, h, rot, seed], dtype=np.float64)
            np.savez_compressed(os.path.join(GOLDEN, f"{name}.npz"), **fx)
            print(name, fx["level_counts"].tolist(), int(fx["floor_fallback"]), int(fx["floor_near"]))
        np.savez_compressed(os.path.join(GOLDEN, "stack3_5mp.npz"),
                            **stack_fixture(2592, 1944, 0, BIG_STRIDE))
        print("stack3_5mp done")
        return
    for name, w, h, rot, seed in SCENES:
        fx = scene_fixture(hf, w, h, rot, seed)
        fx["scene"] = np.array([w, h, rot, seed], dtype=np.float64)
        np.savez_compressed(os.path.join(GOLDEN, f"{name}.npz"), **fx)
        print(name, fx["level_counts"].tolist())
    # error-parity case: the reference's default SceneSpec does not register
    from hdrflow import pipeline
    st = synth.synth_stack(synth.SceneSpec(), 0)
    try:
        pipeline.register_and_fuse(st.ref, st.src)
        raised = ""
    except pipeline.RegistrationError as exc:
        raised = str(exc)
    np.savez_compressed(os.path.join(GOLDEN, "default_scene_error.npz"),
                        inputs_digest=np.array([digest(st.ref), digest(st.src)]),
                        message=np.array(raised))
    print("default scene:", raised)
    np.savez_compressed(os.path.join(GOLDEN, "formats.npz"), **format_fixture())
    np.savez_compressed(os.path.join(GOLDEN, "metering.npz"), **metering_fixture())
    np.savez_compressed(os.path.join(GOLDEN, "stack3_vga.npz"), **stack_fixture(640, 480, 7))
    for name, mode, exposures, swap in FILE_CASES:
        fx = file_fixture(name, mode, exposures, swap)
        np.savez_compressed(os.path.join(GOLDEN, f"{name}.npz"), **fx)
        print(name, fx["level_counts"].tolist())
    # SeedSequence / Philox / choice vectors (weeding.py:62-84)
    rng = np.random.default_rng(7)
    cases = []
    for _ in range(40):
        seed = int(rng.integers(0, 2 ** 32))
        it = int(rng.integers(0, 256))
        n = int(rng.integers(4, 2000))
        ss = np.random.SeedSequence(entropy=seed, spawn_key=(it,))
        key = ss.generate_state(2, np.uint64)
        g = np.random.Generator(np.random.Philox(ss))
        draws = np.stack([g.choice(n, size=4, replace=False) for _ in range(10)])
        cases.append((seed, it, n, key, draws))
    np.savez_compressed(os.path.join(GOLDEN, "philox_choice.npz"),
                        seed=np.array([c[0] for c in cases], dtype=np.uint64),
                        it=np.array([c[1] for c in cases]), n=np.array([c[2] for c in cases]),
                        key=np.stack([c[3] for c in cases]),
                        draws=np.stack([c[4] for c in cases]),
                        level_seeds=np.array([[int(np.random.SeedSequence(entropy=s, spawn_key=(l,))
                                                   .generate_state(1)[0]) for l in range(5)]
                                              for s in (0, 1, 12345, 2 ** 40 + 3)],
                                             dtype=np.uint64))


if __name__ == "__main__":
    main()
