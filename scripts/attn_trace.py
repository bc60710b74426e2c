"""Phase timeline of one FMHA CTA (build with scripts/build_variant.sh
attn_trace -DDM_ATTN_TRACE, run with DM_LIB=_variants/attn_trace.so):
cycles since CTA start of each softmax phase per key block and tile, and of
the MMA warp's S / PV issues."""
import ctypes as C, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model
from paper_2507_01021_b200 import _native

E = 12
eng = WhisperGPU(get_model(sys.argv[1] if len(sys.argv) > 1 else "whisper-large-v3"),
                 max_slots=E, max_encode_batch=E)
rng = np.random.default_rng(0)
segs = [rng.integers(-8000, 8000, size=480000, dtype=np.int16) for _ in range(E)]
for _ in range(2):
    eng.encode(segs, list(range(E)))
torch.cuda.synchronize()
buf = (C.c_ulonglong * 193)()
assert _native.load().dm_attn_trace_read(buf) == 0
a = np.array(buf[:], dtype=np.int64)
t0 = a[192]
sm = a[:128].reshape(2, 16, 4) - t0
mm = a[128:192].reshape(2, 16, 2) - t0
print("tile j | s_full  ld  off  emit | S_issue PV_issue   (cycles since CTA start)")
for j in range(12):
    for t in range(2):
        print(t, j, "|", " ".join(f"{x:6d}" for x in sm[t, j]), "|", " ".join(f"{x:6d}" for x in mm[t, j]))
