"""n-frame stacks (BASELINE config "5MP three-exposure
stack (-2/0/+2 EV) with deghosting and merge").

The reference fuses exactly two frames; the k-way blend is composed from its
own functions. CPU tests pin the oracle's composition against that
composition run on the REAL reference (tests/golden/stack3_vga.npz) and
against the reference's two-frame fuse; GPU tests hold the device path to the
oracle."""

import numpy as np
import pytest

from golden_util import digest, load, scene_inputs
from oracle import gen_golden as G
from oracle import hdr_oracle as O


@pytest.mark.parametrize("name", ["stack3_vga", "stack3_5mp"])
def test_oracle_stack_matches_reference_composition(name):
    """stack3_5mp is BASELINE config C3 at full size (2592x1944)."""
    fx = load(name)
    w, h, seed = (int(v) for v in fx["scene"])
    frames, exposures = G.stack_frames(w, h, seed)
    comp, k, regs = O.register_and_fuse_stack(frames, exposures)
    assert k == int(fx["reference_index"])
    for i, r in enumerate(regs):
        assert r.level_counts == [tuple(x) for x in fx[f"level_counts_{i}"].tolist()]
    assert digest(comp) == str(fx["composite_digest"])


def test_oracle_fuse_stack_of_two_is_fuse():
    fx = load("qvga_s2")
    ref, src = scene_inputs(fx)
    r = O.register_and_fuse(ref, src)
    two = O.fuse_stack([ref, r.warped], [r.ssim], [r.valid.astype(np.float32)])
    assert digest(two) == str(fx["composite_digest"])


@pytest.mark.gpu
def test_stack3_gpu_matches_oracle():
    from paper_1504_01441_b200 import pipeline
    frames, exposures = G.stack_frames(640, 480, 7)
    comp, k, regs = O.register_and_fuse_stack(frames, exposures)
    res = pipeline.register_and_fuse_stack(frames, exposures)
    assert res.reference_index == k
    for got, want in zip(res.registrations, regs):
        assert got.level_counts == want.level_counts
        np.testing.assert_array_equal(got.matches[:, :4], want.matches[:, :4])
        assert np.abs(got.warped - want.warped).max() < 1e-3
        assert got.composite is None
    assert np.abs(res.composite - comp).max() < 1e-3


@pytest.mark.gpu
def test_fuse_stack_two_frames_equals_fuse_and_four_frames(cuda):
    """hdr_fuse_stack with n = 2 is the pair fuse; n = 4 against the oracle
    with synthetic SSIM/validity maps (odd sizes exercise reflect edges)."""
    from paper_1504_01441_b200 import fusion, pipeline
    rng = np.random.default_rng(5)
    h, w = 131, 203
    fr = [rng.random((h, w, 3), dtype=np.float32) for _ in range(4)]
    ss = [rng.uniform(-0.2, 1.0, (h, w)) for _ in range(3)]
    vs = [(rng.random((h, w)) > 0.1) for _ in range(3)]
    two = pipeline.fuse_stack(fr[:2], ss[:1], vs[:1])
    np.testing.assert_array_equal(two, fusion.fuse(fr[0], fr[1], ss[0].astype(np.float32), vs[0]))
    assert np.abs(two - O.fuse(fr[0], fr[1], ss[0].astype(np.float32), vs[0].astype(np.float32))).max() < 1e-3
    for n in (3, 4):
        got = pipeline.fuse_stack(fr[:n], ss[:n - 1], vs[:n - 1])
        want = O.fuse_stack(fr[:n], [s.astype(np.float32) for s in ss[:n - 1]],
                            [v.astype(np.float32) for v in vs[:n - 1]])
        assert np.abs(got - want).max() < 1e-3, n
    with pytest.raises(ValueError):
        pipeline.fuse_stack(fr[:1], [], [])


@pytest.mark.gpu
@pytest.mark.slow
def test_stack3_5mp_gpu_matches_oracle():
    """BASELINE config C3 at full size: -2/0/+2 EV 5MP stack."""
    from paper_1504_01441_b200 import pipeline
    frames, exposures = G.stack_frames(2592, 1944, 0)
    comp, k, regs = O.register_and_fuse_stack(frames, exposures)
    res = pipeline.register_and_fuse_stack(frames, exposures)
    assert res.reference_index == k
    for got, want in zip(res.registrations, regs):
        assert got.level_counts == want.level_counts
    assert np.abs(res.composite - comp).max() < 1e-3


@pytest.mark.gpu
def test_stack_errors(cuda):
    """Shape / count errors as ValueError / ConfigError; a source frame that
    cannot register raises RegistrationError like the pairwise reference."""
    from paper_1504_01441_b200 import pipeline
    from harness import synth
    from paper_1504_01441_b200.errors import ConfigError, RegistrationError
    st = synth.synth_stack(synth.working_spec(320, 240), 1)
    with pytest.raises(ValueError):
        pipeline.register_and_fuse_stack([st.ref])
    with pytest.raises(ConfigError):
        pipeline.register_and_fuse_stack([st.ref, st.src[:200]])
    flat = np.full_like(st.ref, 0.5)  # as the reference: no corners, nothing registers
    with pytest.raises(RegistrationError):
        pipeline.register_and_fuse_stack([st.ref, st.src, flat], [4.0, 2.0, 1.0])
    res = pipeline.register_and_fuse_stack([st.src, st.ref], [4.0, 1.0])
    assert res.reference_index == 1 and len(res.registrations) == 1
