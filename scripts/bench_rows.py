"""Active-row histogram of one bench step (the bench's own workload and engine
settings): how many decode steps run at each active-row count.
Usage: python scripts/bench_rows.py"""
import collections, json, sys
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2507_01021_b200.engine import ResidentPCM, SegmentJob, WhisperGPU
from paper_2507_01021_b200.models import get_model


dims = get_model(bench.MODEL)
segs = bench.make_workload(64, 0)
eng = WhisperGPU(dims, seed=0, max_slots=64, max_encode_batch=12, first_encode_batch=12,
                 overlap_encode=True)
flat = np.concatenate([x for _, x in segs])
pcm_dev = torch.from_numpy(flat).to("cuda")
eng.set_resident(pcm_dev)
offs = np.cumsum([0] + [len(x) for _, x in segs[:-1]])
jobs = lambda: [SegmentJob(uid, ResidentPCM(int(o), len(x)), bench.token_cap(len(x) / 16000.0))
                for (uid, x), o in zip(segs, offs)]
eng.run_jobs(jobs())
rows = {"n": 0}
hist = collections.Counter()
real_set, real_step = eng.set_active, eng.step
def set_active(slots):
    rows["n"] = len(slots)
    return real_set(slots)
def step(n):
    hist[rows["n"]] += n
    return real_step(n)
eng.set_active, eng.step = set_active, step
eng.run_jobs(jobs())
torch.cuda.synchronize()
print(json.dumps({"steps": sum(hist.values()), "rows_hist": dict(sorted(hist.items()))}))
