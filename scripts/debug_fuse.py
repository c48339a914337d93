import sys, numpy as np
sys.path.insert(0, '.')
from paper_1504_01441_b200 import pipeline, fusion, synth
from oracle import hdr_oracle as O
st = synth.synth_stack(synth.working_spec(640, 480), 0)
res = pipeline.register_and_fuse(st.ref, st.src)
o = O.register_and_fuse(st.ref, st.src)
c1 = fusion.fuse(st.ref, res.warped, res.ssim, res.valid.astype(np.float32))
c2 = O.fuse(st.ref, res.warped, res.ssim, res.valid.astype(np.float32))
print("pipeline vs oracle", np.abs(res.composite - o.composite).max())
print("stage fuse(gpu inputs) vs pipeline", np.abs(c1 - res.composite).max())
print("stage fuse vs oracle fuse (gpu inputs)", np.abs(c1 - c2).max())
print("oracle fuse(gpu inputs) vs oracle", np.abs(c2 - o.composite).max())
print("ssim", np.abs(res.ssim - o.ssim).max(), "warped", np.abs(res.warped - o.warped).max(), "valid", (res.valid != o.valid).sum())
res2 = pipeline.register_and_fuse(st.ref, st.src)
print("pipeline repeat identical", np.array_equal(res2.composite, res.composite))
bad = np.argwhere(np.abs(res.composite - o.composite).max(axis=2) > 1e-3)
print("bad pixels", len(bad), bad[:10])
