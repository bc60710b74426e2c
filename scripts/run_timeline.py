"""Kernel timeline of one bench step (torch.profiler / CUPTI activity, not
ncu): per kernel family the summed device time, the encode / decode split
and how much of the step each stream kept busy. Usage:
python scripts/run_timeline.py [first_encode_batch] [encode_batch]"""
import collections, json, sys
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2507_01021_b200.engine import ResidentPCM, SegmentJob, WhisperGPU
from paper_2507_01021_b200.models import get_model

fe = int(sys.argv[1]) if len(sys.argv) > 1 else 24
eb = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dims = get_model(bench.MODEL)
segs = bench.make_workload(64, 0)
import os
eng = WhisperGPU(dims, max_slots=64, max_encode_batch=eb, first_encode_batch=fe,
                 length_aware=bool(int(os.environ.get("LA", "0"))))
flat = np.concatenate([x for _, x in segs])
pcm = torch.from_numpy(flat).cuda()
eng.set_resident(pcm)
offs = np.cumsum([0] + [len(x) for _, x in segs[:-1]])
jobs = lambda: [SegmentJob(u, ResidentPCM(int(o), len(x)), bench.token_cap(len(x) / 16000.0))
                for (u, x), o in zip(segs, offs)]
for _ in range(3):
    eng.run_jobs(jobs())
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.run_jobs(jobs())
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.device_time_total > 0]
ks = []
for e in ev:
    name = e.name.split("(")[0].replace("void ", "")
    ks.append((e.time_range.start, e.time_range.end, name))
ks.sort()
t0, t1 = ks[0][0], max(k[1] for k in ks)
enc_names = ("gemm", "attn_tcgen05", "logmel", "layernorm_bf16")
fam = collections.defaultdict(float)
enc_iv, dec_iv = [], []
for s, e, n in ks:
    fam[n.split("<")[0]] += (e - s)
    (enc_iv if any(k in n for k in enc_names) else dec_iv).append((s, e))
def union(iv):
    iv = sorted(iv); tot = 0; cs, ce = None, None
    for s, e in iv:
        if cs is None or s > ce:
            if cs is not None: tot += ce - cs
            cs, ce = s, e
        else: ce = max(ce, e)
    if cs is not None: tot += ce - cs
    return tot
first_dec = min(s for s, _ in dec_iv) if dec_iv else None
last_enc = max(e for _, e in enc_iv)
out = {"step_ms": (t1 - t0) / 1e3, "first_encode_batch": fe, "encode_batch": eb,
       "encode_busy_ms": union(enc_iv) / 1e3, "decode_busy_ms": union(dec_iv) / 1e3,
       "any_busy_ms": union(enc_iv + dec_iv) / 1e3,
       "first_decode_at_ms": (first_dec - t0) / 1e3, "last_encode_end_ms": (last_enc - t0) / 1e3,
       "families_ms": {k: round(v / 1e3, 2) for k, v in sorted(fam.items(), key=lambda kv: -kv[1])[:14]}}
print(json.dumps(out, indent=1))
