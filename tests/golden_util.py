"""Helpers shared by the oracle/golden and GPU parity tests."""
import hashlib
import os

import numpy as np

from harness import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SCENES = ["vga_s0", "vga_rot_s1", "qvga_s2", "r960_s3"]
# BASELINE configs[1] (5MP) and configs[3] (12MP), from the real reference
BIG_SCENES = ["c2_5mp_s0", "c4_12mp_s0"]
# rows wider than the shared-memory row kernels (7200 px), same fixture format
WIDE_SCENES = ["wide_7200x1000_s0"]


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()


def load(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))


def scene_inputs(fx):
    w, h, rot, seed = fx["scene"]
    st = synth.synth_stack(synth.working_spec(int(w), int(h), rotation_deg=float(rot)), int(seed))
    return st.ref, st.src
