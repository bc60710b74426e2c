"""Stress test for the experimental overlapped encode: runs
WhisperGPU.run_jobs on the bench workload REPS times with overlap_encode on
and checks every run's tokens against a serial run.
usage: python scripts/overlap_repro.py SEGMENTS FIRST ENCODE_BATCH REPS [ENC_LAYERS]"""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import MODEL, make_workload, token_cap
from paper_2507_01021_b200.engine import ResidentPCM, SegmentJob, WhisperGPU
from paper_2507_01021_b200.models import get_model

n, first, eb, reps = map(int, sys.argv[1:5])
segs = make_workload(n)
eng = WhisperGPU(get_model(MODEL), seed=0, device=0, max_slots=min(64, n), max_encode_batch=eb,
                 first_encode_batch=first)
pcm = torch.from_numpy(np.concatenate([x for _, x in segs])).cuda()
eng.set_resident(pcm)
offs = np.cumsum([0] + [len(x) for _, x in segs[:-1]])
jobs = lambda: [SegmentJob(u, ResidentPCM(int(o), len(x)), token_cap(len(x) / 16000.0))
                for (u, x), o in zip(segs, offs)]
if len(sys.argv) > 5:            # debug: run only the first ENC_LAYERS encoder layers
    eng.lib.dm_whisper_debug(eng.handle, 4, None, int(sys.argv[5]), eng._s)
guard = np.zeros(64, np.int32)


def check(tag):
    if eng.lib.dm_whisper_debug(eng.handle, 13, guard.ctypes.data_as(C.c_void_p), guard.nbytes,
                                eng._s) == 0 and guard[0]:
        print(f"GUARD {tag}: {guard[0]} bad, (index, offset, KB) {guard[1:1 + 3 * guard[0]].tolist()}",
              flush=True)


ref = eng.run_jobs(jobs())
torch.cuda.synchronize()
check("serial")
eng.overlap_encode = True
for i in range(reps):
    t = time.perf_counter()
    try:
        out = eng.run_jobs(jobs())
        torch.cuda.synchronize()
    except Exception as ex:
        print(f"FAIL n={n} first={first} eb={eb} run={i}: {str(ex).splitlines()[0]}", flush=True)
        raise SystemExit(1)
    check(f"run {i}")
    same = all(out[k] == ref[k] for k in ref)
    print(f"ok n={n} first={first} eb={eb} run={i} same={same} "
          f"{1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
