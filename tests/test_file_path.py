"""File path (SURVEY.md §8(f)1 + (f)3): PNG ingest, reference choice,
8-bit output, stage-dump formats.

CPU tests pin the oracle's run_hdr against the real reference's outputs
(tests/golden/file_*.npz, made by oracle/gen_golden.py) and the dump writers
against the reference's bytes; GPU tests hold the device path to the oracle."""

import os

import numpy as np
import pytest

from golden_util import digest, load
from oracle import gen_golden as G
from oracle import hdr_oracle as O

FILE_CASES = [c[0] for c in G.FILE_CASES]


def case_files(tmp_path, name):
    fx = load(name)
    paths = G.write_scene_pngs(str(tmp_path), str(fx["mode"]), bool(fx["swap"]))
    return fx, paths, [float(e) for e in fx["exposures"]]


@pytest.mark.parametrize("name", FILE_CASES)
def test_oracle_run_hdr_matches_reference(tmp_path, name):
    fx, paths, exposures = case_files(tmp_path, name)
    imgs = [O.load_png(p) for p in paths]
    assert [digest(a) for a in imgs] == list(fx["inputs_digest"])
    out, comp8, _ = O.run_hdr(paths, exposures)
    assert out.level_counts == [tuple(x) for x in fx["level_counts"].tolist()]
    assert digest(out.composite) == str(fx["composite_digest"])
    assert digest(comp8) == str(fx["composite_u8_digest"])


def test_raw_reader_matches_load_png(tmp_path):
    """read_png_raw keeps the samples load_png scales (host side, no GPU)."""
    from PIL import Image
    from paper_1504_01441_b200 import fileio
    rng = np.random.default_rng(3)
    rgb = rng.integers(0, 256, (9, 11, 3), dtype=np.uint8)
    cases = {"RGB": Image.fromarray(rgb, "RGB"), "L": Image.fromarray(rgb[..., 0], "L"),
             "RGBA": Image.fromarray(np.dstack([rgb, rgb[..., :1]]), "RGBA"),
             "P": Image.fromarray(rgb, "RGB").convert("P"),
             "I;16": Image.fromarray(rng.integers(0, 65536, (9, 11), dtype=np.uint16), "I;16")}
    for mode, im in cases.items():
        path = os.path.join(tmp_path, f"{mode.replace(';', '_')}.png")
        im.save(path, format="PNG")
        raw, bits = fileio.read_png_raw(path)
        want = O.load_png(path)
        got = np.clip(raw.astype(np.float64) / (65535.0 if bits == 16 else 255.0), 0, 1).astype(np.float32)
        np.testing.assert_array_equal(got, want, err_msg=mode)
    bad = os.path.join(tmp_path, "bad.png")
    open(bad, "wb").write(b"not a png")
    with pytest.raises(fileio.FileFormatError):
        fileio.read_png_raw(bad)


def test_harmonize_raw_is_exact():
    """8 -> 16 bit by x257 and grey -> RGB leave load_png's values unchanged."""
    from paper_1504_01441_b200.pipeline import harmonize_raw
    v8 = np.arange(256, dtype=np.uint8).reshape(16, 16)
    v16 = np.zeros((16, 16, 3), dtype=np.uint16)
    (a, b), bits = harmonize_raw([(v8, 8), (v16, 16)])
    assert bits == 16 and a.shape == (16, 16, 3) and b.shape == (16, 16, 3)
    f8 = (v8.astype(np.float64) / 255.0).astype(np.float32)
    f16 = (a[..., 0].astype(np.float64) / 65535.0).astype(np.float32)
    np.testing.assert_array_equal(f8, f16)


def test_dump_formats_match_reference_bytes(tmp_path):
    from paper_1504_01441_b200 import fileio
    fx = load("formats")
    for name, fn in (("grey", fileio.save_pfm), ("colour", fileio.save_pfm),
                     ("matches", fileio.save_matches_csv)):
        path = os.path.join(tmp_path, name)
        fn(path, fx[name])
        assert open(path, "rb").read() == fx[f"{name}_bytes"].tobytes(), name
    np.testing.assert_array_equal(fileio.load_pfm(os.path.join(tmp_path, "grey")), fx["grey"])
    np.testing.assert_array_equal(fileio.load_pfm(os.path.join(tmp_path, "colour")), fx["colour"])
    np.testing.assert_array_equal(fileio.load_matches_csv(os.path.join(tmp_path, "matches")),
                                  fx["matches"])
    side = os.path.join(tmp_path, "exp.txt")
    open(side, "w").write("# sidecar\na b.png 0.5\n\nc.png 2\n")
    assert fileio.load_exposures(side) == [("a b.png", 0.5), ("c.png", 2.0)]
    open(side, "w").write("lonely\n")
    with pytest.raises(fileio.FileFormatError):
        fileio.load_exposures(side)


def test_resolve_exposures_mirror(tmp_path):
    from paper_1504_01441_b200.errors import ConfigError
    from paper_1504_01441_b200.pipeline import PipelineConfig, _resolve_exposures
    assert _resolve_exposures(PipelineConfig(inputs=["a", "b"])) == (["a", "b"], [1.0, 1.0])
    assert _resolve_exposures(PipelineConfig(inputs=["a", "b"], exposures=[2, 1])) == (["a", "b"], [2, 1])
    with pytest.raises(ConfigError):
        _resolve_exposures(PipelineConfig(inputs=["a", "b"], exposures=[1]))
    side = os.path.join(tmp_path, "e.txt")
    open(side, "w").write("x.png 1\ny.png 3\n")
    assert _resolve_exposures(PipelineConfig(exposure_file=side)) == (["x.png", "y.png"], [1.0, 3.0])
    with pytest.raises(ConfigError):
        _resolve_exposures(PipelineConfig(inputs=["z.png"], exposure_file=side))


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", FILE_CASES)
def test_run_hdr_gpu(tmp_path, name):
    """pipeline.run_hdr on the GPU: same reference choice and level counts as
    the oracle, PNG output within 1 LSB (the f32 fusion moves a few pixels
    across a quantisation boundary), f32 composite <= 1e-3."""
    from PIL import Image
    from paper_1504_01441_b200 import pipeline
    fx, paths, exposures = case_files(tmp_path, name)
    outp = os.path.join(tmp_path, "out.png")
    res = pipeline.run_hdr(pipeline.PipelineConfig(inputs=paths, exposures=exposures, output=outp))
    ora, comp8, _ = O.run_hdr(paths, exposures)
    assert res.level_counts == ora.level_counts
    np.testing.assert_array_equal(res.matches[:, :4], ora.matches[:, :4])
    assert np.abs(res.composite - ora.composite).max() < 1e-3
    with Image.open(outp) as im:
        got8 = np.asarray(im)
    d = np.abs(got8.astype(int) - comp8.astype(int))
    assert d.max() <= 1 and (d > 0).mean() < 1e-3


@pytest.mark.gpu
def test_decode_encode_mean_bit_exact(tmp_path):
    import torch
    from paper_1504_01441_b200 import fileio, metering
    from paper_1504_01441_b200.pipeline import harmonize_raw
    rng = np.random.default_rng(9)
    for bits, shape in ((8, (33, 47, 3)), (8, (33, 47)), (16, (20, 31, 3)), (16, (20, 31))):
        raw = rng.integers(0, 2 ** bits, shape).astype(np.uint8 if bits == 8 else np.uint16)
        rgb = fileio.decode_rgb(fileio.raw_to_device(raw, bits), bits).cpu().numpy()
        want = O.as_rgb(np.clip(raw.astype(np.float64) / (2.0 ** bits - 1), 0, 1).astype(np.float32))
        np.testing.assert_array_equal(rgb, want)
        np.testing.assert_array_equal(fileio.quantize_u8(rgb).cpu().numpy(), O.png_quantize(rgb))
        m = metering.mean_luminance(torch.from_numpy(rgb).cuda())
        assert abs(m - float(np.mean(O.luminance(rgb)))) < 1e-6
    edge = np.array([-0.5, 0.0, 0.5 / 255, 1.5 / 255, 0.999, 1.0, 7.0, np.nan], dtype=np.float32)
    np.testing.assert_array_equal(fileio.quantize_u8(edge[:7]).cpu().numpy(), O.png_quantize(edge[:7]))
    (a, b), bits = harmonize_raw([(np.arange(256, dtype=np.uint8).reshape(16, 16), 8),
                                  (np.zeros((16, 16), np.uint16), 16)])
    got = fileio.decode_rgb(fileio.raw_to_device(a, bits), bits).cpu().numpy()
    np.testing.assert_array_equal(got[..., 0], (np.arange(256).reshape(16, 16) / 255.0).astype(np.float32))


@pytest.mark.gpu
def test_choose_reference_and_dumps(tmp_path):
    from paper_1504_01441_b200 import fileio, metering, pipeline
    fx, paths, _ = case_files(tmp_path, "file_rgb8_tie")
    imgs = [O.as_rgb(O.load_png(p)) for p in paths]
    assert metering.choose_reference(imgs, [2.0, 2.0]) == O.choose_reference(imgs, [2.0, 2.0])
    assert metering.choose_reference(imgs, [3.0, 2.0]) == 1
    with pytest.raises(ValueError):
        metering.choose_reference(imgs, [1.0])
    d = os.path.join(tmp_path, "dump")
    res = pipeline.run_hdr(pipeline.PipelineConfig(inputs=paths, exposures=[2.0, 2.0],
                                                   output=os.path.join(tmp_path, "o.png"),
                                                   dump_all=True, out_dir=d))
    names = sorted(os.listdir(d))
    assert names == sorted(["matches_raw.csv", "matches.csv", "matches.png", "flow.pfm", "flow.png",
                            "warped.pfm", "warped.png", "valid.pfm", "ssim.pfm", "ssim.png",
                            "weight_ref.pfm", "weight_src.pfm", "weight_ref.png", "weight_src.png"])
    np.testing.assert_array_equal(fileio.load_matches_csv(os.path.join(d, "matches.csv")), res.matches)
    np.testing.assert_array_equal(pipeline.pfm_to_flow(fileio.load_pfm(os.path.join(d, "flow.pfm"))),
                                  res.flow)
    k = O.choose_reference(imgs, [2.0, 2.0])
    wr, ws = O.fusion_weights(imgs[k], res.warped, res.ssim, res.valid.astype(np.float32))
    assert np.abs(fileio.load_pfm(os.path.join(d, "weight_src.pfm")) - ws).max() < 1e-5
    assert np.abs(fileio.load_pfm(os.path.join(d, "weight_ref.pfm")) - wr).max() < 1e-5


def test_flow_to_color_per_pixel():
    """viz.flow_to_color = the per-pixel hue-sector colouring the reference
    intends (its fancy-indexing form would gather (h, w, h, w); see viz.py),
    checked against the reference's six-entry ramp evaluated per pixel."""
    from paper_1504_01441_b200 import viz
    f = np.random.default_rng(0).normal(size=(5, 6, 2)).astype(np.float32)
    got = viz.flow_to_color(f)
    u, v = f[..., 0].astype(np.float64), f[..., 1].astype(np.float64)
    mag = np.minimum(np.hypot(u, v) / np.hypot(u, v).max(), 1.0)
    h6 = (np.arctan2(-v, -u) / np.pi + 1.0) / 2.0 * 6.0
    for i in range(5):
        for j in range(6):
            s = min(int(h6[i, j]), 5)
            t = h6[i, j] - s
            ramp = [1.0, 1.0 - t, 0.0, 0.0, t, 1.0]
            rgb = np.array([ramp[s % 6], ramp[(s + 4) % 6], ramp[(s + 2) % 6]])
            np.testing.assert_allclose(got[i, j], (1.0 - mag[i, j] * (1.0 - rgb)).astype(np.float32),
                                       atol=1e-6)
    hm = viz.heatmap(np.array([[-1.0, 0.0, 1.0]]), -1.0, 1.0)
    np.testing.assert_array_equal(hm[0], np.array([[0, 0, 1], [1, 1, 1], [1, 0, 0]], dtype=np.float32))
    x = np.random.default_rng(1).random((4, 5))
    t = x
    ref_rgb = np.stack([np.clip(2 * t, 0, 1), 1 - np.abs(2 * t - 1), np.clip(2 * (1 - t), 0, 1)], -1)
    np.testing.assert_allclose(viz.heatmap(x, 0.0, 1.0), ref_rgb.astype(np.float32), atol=1e-6)


def test_overlay_matches_segments():
    """Every pixel the reference's per-match line walk (viz.py:44-58) paints
    is painted, in green for the displacement and red at the reference end."""
    from paper_1504_01441_b200 import viz
    lum = np.full((40, 50), 0.5, dtype=np.float32)
    m = np.array([[3.0, 4.0, 20.0, 9.0, 0.1], [45.0, 30.0, 60.0, 35.0, 0.2]])
    got = viz.overlay_matches(lum, m)
    canvas = np.repeat(lum[:, :, None], 3, axis=2).copy()
    for xr, yr, xs, ys, _ in m:
        n = int(max(abs(xs - xr), abs(ys - yr))) + 1
        px, py = np.round(np.linspace(xr, xs, n)).astype(int), np.round(np.linspace(yr, ys, n)).astype(int)
        ok = (px >= 0) & (px < 50) & (py >= 0) & (py < 40)
        canvas[py[ok], px[ok]] = (0.1, 0.9, 0.2)
    for xr, yr, _, _, _ in m:
        canvas[int(yr), int(xr)] = (1.0, 0.2, 0.1)
    np.testing.assert_array_equal(got, canvas.astype(np.float32))


@pytest.mark.gpu
def test_run_hdr_errors(tmp_path):
    from paper_1504_01441_b200 import pipeline
    from paper_1504_01441_b200.errors import ConfigError
    _, paths, _ = case_files(tmp_path, "file_rgb8")
    with pytest.raises(ConfigError):
        pipeline.run_hdr(pipeline.PipelineConfig(inputs=paths[:1]))
    with pytest.raises(ConfigError):
        pipeline.run_hdr(pipeline.PipelineConfig(inputs=paths, exposures=[1.0]))
    with pytest.raises(ConfigError):
        pipeline.run_hdr(pipeline.PipelineConfig(inputs=paths, params=pipeline.PipelineParams(tile=8)))
    with pytest.raises(FileNotFoundError):
        pipeline.run_hdr(pipeline.PipelineConfig(inputs=[paths[0], str(tmp_path / "missing.png")]))


def test_oracle_metering_matches_reference():
    fx = load("metering")
    imgs = G.metering_images()
    assert [O.select_offset(x) for x in imgs] == fx["offsets"].tolist()
    plans = [list(O.plan_stack([imgs[i], imgs[i + 2]], [1.0, 1.0])) for i in range(0, 6, 2)]
    assert plans == fx["plans"].tolist()


@pytest.mark.gpu
def test_metering_gpu_matches_oracle():
    from paper_1504_01441_b200 import metering
    imgs = G.metering_images()
    for x in imgs:
        assert metering.select_offset(x) == O.select_offset(x)
        lum = O.luminance(x) if x.ndim == 3 else x
        assert metering.dark_fraction(x) == float(np.mean(lum < 0.05))
        assert abs(metering.mean_luminance(x) - float(np.mean(lum))) < 1e-6
    for i in range(0, 6, 2):
        p = metering.plan_stack([imgs[i], imgs[i + 2]], [1.0, 1.0])
        assert (p.offset_stops, p.reference_index) == O.plan_stack([imgs[i], imgs[i + 2]], [1.0, 1.0])
