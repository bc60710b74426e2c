"""Decode-step timeline from in-kernel globaltimer marks (debug tap 10-12):
per kernel of the step graph, the dependency-release time (first CTA past
griddepcontrol.wait) relative to the previous kernel's last exit, and its own
release-to-exit span. Usage: python scripts/step_trace.py [model] [rows...]"""
import ctypes as C, json, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model

name = sys.argv[1] if len(sys.argv) > 1 else "whisper-base"
rows_list = [int(x) for x in sys.argv[2:]] or [64, 32, 8, 1]
dims = get_model(name)
S = 64
import os
eng = WhisperGPU(dims, max_slots=S, max_encode_batch=32,
                 length_aware=bool(int(os.environ.get("LA", "0"))))

rng = np.random.default_rng(0)
seg = rng.integers(-8000, 8000, size=160000, dtype=np.int16)
slots = list(range(S))
for i in range(0, S, 32):
    eng.encode([seg] * 32, slots[i:i + 32])
eng.admit(slots, [400] * S)
XA_TAIL_MERGE_ROWS = int(os.environ.get("DM_XA_TAIL_MERGE_ROWS", "0"))  # kXaTailMergeRows
FC1_TAIL_ROWS = int(os.environ.get("DM_FC1_TAIL_ROWS", "0"))
GV_FUSE_ROWS = min(16, int(os.environ.get("DM_GV_FUSE_ROWS", "8")))     # kGvFuseRows


def names_for(rows):
    names = []
    fuse = rows <= GV_FUSE_ROWS
    for l in range(dims.dec_layers):
        kinds = ["ln1", "qkv", "self", "o", "ln2", "xq", "xattn"]
        if rows > XA_TAIL_MERGE_ROWS and not fuse:           # split merge kernel
            kinds.append("xmerge")
        kinds += ["xo", "ln3", "fc1"]
        if dims.d_model // 64 > 8 and rows > FC1_TAIL_ROWS and not fuse:   # GELU kernel
            kinds.append("gelu")
        kinds.append("fc2")
        names += [f"L{l}.{k}" for k in kinds]
    lm = ["lm_head"] if os.environ.get("DM_LM_ARGMAX_EPI") else ["lm_head", "lm_argmax"]
    return names + ["ln_f"] + lm + ["finalize"]
lib = eng.lib
def dbg(which, buf=None, n=0):
    ptr = buf.ctypes.data_as(C.c_void_p) if buf is not None else None
    from paper_2507_01021_b200 import _native
    _native.check(lib.dm_whisper_debug(eng.handle, which, ptr, buf.nbytes if buf is not None else n, eng._s))
dbg(10)
out = {}
for rows in rows_list:
    names = names_for(rows)
    eng.set_active(slots[:rows])
    eng.step(6)
    torch.cuda.synchronize()
    acc = None
    reps = 10
    for _ in range(reps):
        dbg(11)
        eng.step(1)
        torch.cuda.synchronize()
        t = np.zeros((512, 8), np.uint64)
        dbg(12, t)
        t = t[:len(names)].astype(np.float64)
        t0 = t[0, 1]
        t = t - t0
        acc = t if acc is None else acc + t
    t = acc / reps
    res = []
    prev_end = 0.0
    for k, nm in enumerate(names):
        entry, rel, rel_max, end = t[k][:4]
        rec = {"k": nm, "gap_us": round((rel - prev_end) / 1e3, 2),
               "span_us": round((end - rel) / 1e3, 2),
               "early_us": round((rel - entry) / 1e3, 2),
               "rel_spread_us": round((rel_max - rel) / 1e3, 2)}
        kind = nm.split(".")[-1]
        labs = {"self": ((4, "qkv_ready"), (5, "pages_landed"), (6, "softmax_done"), (7, "pv_done")),
                "ln1": ((4, "loaded"), (5, "stats_done")), "ln2": ((4, "loaded"), (5, "stats_done")),
                "ln3": ((4, "loaded"), (5, "stats_done")), "ln_f": ((4, "loaded"), (5, "stats_done")),
                "xattn": ((4, "tmem_alloc"), (5, "k_landed"), (6, "s_issued"), (7, "merged")),
                }.get(kind, ((4, "x_landed"), (7, "mma_issued"), (5, "mma_done"), (6, "stores")))
        for j, lab in labs:
            if t[k][j] > 0:
                rec[lab + "_us"] = round((t[k][j] - rel) / 1e3, 2)
        res.append(rec)
        prev_end = end
    total = t[len(names) - 1, 3] / 1e3
    kinds = {}
    for r in res:
        kk = r["k"].split(".")[-1]
        d = kinds.setdefault(kk, [0.0, 0.0, 0])
        d[0] += r["gap_us"]; d[1] += r["span_us"]; d[2] += 1
    out[rows] = {"step_us": round(total, 1),
                 "by_kind": {k: {"n": v[2], "gap_us": round(v[0], 1), "span_us": round(v[1], 1)} for k, v in kinds.items()},
                 "layer0": res[:12]}
print(json.dumps(out, indent=1))
