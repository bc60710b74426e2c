"""Per-phase durations of the persistent decode kernel (globaltimer at each
grid barrier, block 0)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch, json
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model
name = sys.argv[1] if len(sys.argv) > 1 else "whisper-base"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dims = get_model(name)
eng = WhisperGPU(dims, max_slots=64, max_encode_batch=32, persistent_decode=True)
rng = np.random.default_rng(0)
segs = [rng.integers(-8000, 8000, size=160000, dtype=np.int16) for _ in range(32)]
slots = list(range(64))
eng.encode(segs, slots[:32]); eng.encode(segs, slots[32:])
eng.admit(slots, [200] * 64)
eng.set_active(slots[:rows])
eng.debug(8)
eng.step(3)
eng.step(2)
torch.cuda.synchronize()
ts = np.empty(1 << 16, np.uint64)
eng.debug(9, ts)
L = dims.dec_layers
per_step = 1 + 11 * L + 3
names = ["embed"] + [f"L{l}.{p}" for l in range(L) for p in ("ln1", "qkv", "self", "o", "ln2", "xq", "cross", "xo", "ln3", "fc1", "fc2")] + ["lnf", "lmhead", "final"]
d = np.diff(ts[:2 * per_step].astype(np.int64)) / 1000.0
step2 = d[per_step - 1: 2 * per_step - 1]
agg = {}
for n, v in zip(names, step2):
    k = n.split(".")[-1]
    agg[k] = agg.get(k, 0) + v
print(json.dumps({"rows": rows, "step_us": float(step2.sum()), "by_phase_us": {k: round(v, 1) for k, v in agg.items()}}, indent=1))
