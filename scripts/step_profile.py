"""Per-phase timing on one GPU (CUDA events): encoder for a batch of segments
and one decode step (CUDA-graph replay) at several active-slot counts."""
import argparse, json, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="whisper-base")
ap.add_argument("--slots", type=int, default=64)
ap.add_argument("--encode-batch", type=int, default=32)
args = ap.parse_args()
dims = get_model(args.model)
eng = WhisperGPU(dims, max_slots=args.slots, max_encode_batch=args.encode_batch)
rng = np.random.default_rng(0)
segs = [rng.integers(-8000, 8000, size=480000, dtype=np.int16) for _ in range(args.encode_batch)]
ev = lambda: torch.cuda.Event(enable_timing=True)
out = {"model": args.model}
for it in range(3):
    a, b = ev(), ev()
    a.record(eng.stream); eng.encode(segs, list(range(args.encode_batch))); b.record(eng.stream)
    torch.cuda.synchronize()
out["encode_ms_per_batch"] = a.elapsed_time(b)
out["encode_ms_per_segment"] = a.elapsed_time(b) / args.encode_batch
flops = 2*dims.n_mels*3*dims.d_model*3000 + 2*3*dims.d_model**2*1500 + dims.enc_layers*(24*dims.d_model**2*1500 + 4*1500**2*dims.d_model)
flops += 4*dims.dec_layers*dims.d_model**2*1500
out["encoder_tflops"] = flops * args.encode_batch / (a.elapsed_time(b) / 1e3) / 1e12
slots = list(range(args.slots))
for i in range(0, args.slots, args.encode_batch):
    ch = slots[i:i + args.encode_batch]
    eng.encode(segs[:len(ch)], ch)
eng.admit(slots, [400] * args.slots)
res = {}
for n in (64, 48, 32, 16, 8, 1):
    if n > args.slots: continue
    eng.set_active(slots[:n])
    eng.step(4)
    a, b = ev(), ev()
    a.record(eng.stream); eng.step(20); b.record(eng.stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    xkv = n * dims.dec_layers * 2 * 1500 * dims.d_model * 2
    res[n] = {"step_ms": round(ms, 4), "xkv_GBps": round(xkv / ms / 1e6, 1)}
out["decode_step"] = res
names = {0: "cross_attn", 1: "self_attn", 2: "lm_head", 3: "decode_ln", 4: "gemv_xq",
         5: "gemv_fc2", 6: "empty_pdl_floor", 7: "gemv_fc1", 8: "gemv_qkv"}
for n in (64, 1):
    eng.set_active(slots[:n])
    out[f"kernel_us_rows{n}"] = {names[w]: round(1000 * eng.time_kernel(w, 0, 50), 2) for w in names}
print(json.dumps(out, indent=1))
