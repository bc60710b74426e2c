"""Run individual decode-step kernels at a chosen active-row count (for ncu
captures): python scripts/decode_kernel_probe.py ROWS WHICH[,WHICH...] (ids as
dm_whisper_time_kernel: 0 cross-attn, 1 self-attn, 2 LM head, 3 LN, 4 xq,
5 fc2, 7 fc1, 8 qkv)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 64
which = [int(w) for w in (sys.argv[2] if len(sys.argv) > 2 else "0").split(",")]
model = sys.argv[3] if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else "whisper-base"
dims = get_model(model)
eng = WhisperGPU(dims, max_slots=64, max_encode_batch=32)
seg = np.random.default_rng(0).integers(-8000, 8000, size=160000, dtype=np.int16)
slots = list(range(64))
for i in range(0, 64, 32):
    eng.encode([seg] * 32, slots[i:i + 32])
eng.admit(slots, [200] * 64)
eng.set_active(slots[:rows])
if "--nostep" not in sys.argv:
    eng.step(40)
torch.cuda.synchronize()
for w in which:
    us = 1000 * eng.time_kernel(w, 0, 5)
    print(f"kernel {w}: {us:.2f} us (rows {rows})")
