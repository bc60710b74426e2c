"""Host-side profile of the e2e path (SegmentQueue -> B200Backend.transcribe_batch)
on the bench workload: wall time per phase of run_jobs and a cProfile top list."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2507_01021_b200.backend import B200Backend, B200BackendConfig
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model
from paper_2507_01021_b200.types import make_segment

rs = bench.reference_scheduler()
segs = bench.make_workload(64, 0)
eng = WhisperGPU(get_model(bench.MODEL), max_slots=64, max_encode_batch=64, first_encode_batch=24)
backend = B200Backend(B200BackendConfig(model=bench.MODEL), engine=eng)

def once():
    q = rs.SegmentQueue()
    for uid, x in segs:
        q.enqueue_segment(make_segment(uid, x, session_id=uid, endpoint_time=0.0), 0.0)
    pol = rs.BatchingPolicy(kind="continuous", min_batch=32, max_batch=64)
    batch = q.try_form_batch(pol, 0.0)
    return backend.transcribe_batch(batch)

for _ in range(3):
    once()
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter(); once(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print("e2e wall ms", [round(1000 * t, 2) for t in ts])
pr = cProfile.Profile()
pr.enable(); once(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
