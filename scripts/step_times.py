"""Decode step time per active-row count (CUDA events on the engine stream
around 20 back-to-back step-graph replays; no trace marks). Every row count
starts from fresh slots advanced to position POS (default 40), so all are
timed over positions POS..POS+19.
Usage: python scripts/step_times.py [model] [rows...] [--pos POS] [--groups G]"""
import json, statistics, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model

args = [a for a in sys.argv[1:]]
pos, groups = 40, 1
for flag in ("--pos", "--groups"):
    if flag in args:
        i = args.index(flag)
        v = int(args[i + 1])
        del args[i:i + 2]
        if flag == "--pos":
            pos = v
        else:
            groups = v
name = args[0] if args else "whisper-large-v3"
rows_list = [int(x) for x in args[1:]] or [64, 48, 32, 16, 8, 4, 2, 1]
dims = get_model(name)
S = 64
eng = WhisperGPU(dims, max_slots=S, max_encode_batch=32, decode_groups=groups)
seg = np.random.default_rng(0).integers(-8000, 8000, size=160000, dtype=np.int16)
slots = list(range(S))
for i in range(0, S, 32):
    eng.encode([seg] * 32, slots[i:i + 32])
out = {}
for rows in rows_list:
    eng.admit(slots[:rows], [440] * rows)
    eng.set_active(slots[:rows])
    eng.step(pos)
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(eng.stream)
        eng.step(4)
        b.record(eng.stream)
        b.synchronize()
        ts.append(a.elapsed_time(b) / 4)
    eng.release(slots[:rows])
    out[rows] = round(1000 * statistics.median(ts), 1)
    print(rows, out[rows], "us per step", flush=True)
print(json.dumps({"model": name, "pos": pos, "groups": groups, "step_us": out}))
