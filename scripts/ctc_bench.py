#!/usr/bin/env python
"""cfg5 throughput: wav2vec2-base CTC on short, low-padding segments
(U[1, 8] s loadgen-style speech), RTFx = audio-s / device-s with PCM resident
in HBM (CUDA events on the engine stream), plus the CPU oracle on a sample."""
import argparse, json, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_01021_b200.ctc import Wav2Vec2GPU

ap = argparse.ArgumentParser()
ap.add_argument("--segments", type=int, default=256)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--cpu-sample", type=int, default=4)
args = ap.parse_args()
rng = np.random.default_rng(5)
segs = [rng.integers(-8000, 8000, size=int(rng.uniform(1, 8) * 16000), dtype=np.int16)
        for _ in range(args.segments)]
audio = sum(len(s) for s in segs) / 16000
eng = Wav2Vec2GPU(max_batch=args.batch, max_samples=8 * 16000)
flat = np.concatenate(segs)
pcm = torch.from_numpy(flat).cuda()
offs = np.cumsum([0] + [len(s) for s in segs[:-1]]).tolist()

def step():
    for i in range(0, len(segs), args.batch):
        eng.run(segs[i:i + args.batch], resident=(pcm, offs[i:i + args.batch]))
    eng.stream.synchronize()

step(); step()
ts = []
for _ in range(args.steps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(eng.stream); step(); b.record(eng.stream); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = sum(ts) / len(ts)
flops = 13.82e9 * audio
out = {"metric": "CTC RTFx (cfg5, 1 GPU)", "value": audio / (ms / 1e3), "audio_s": audio,
       "segments": args.segments, "ms_per_step": ms, "tflops": flops / (ms / 1e3) / 1e12}
import os
from oracle.wav2vec2 import Wav2Vec2Oracle
torch.set_num_threads(len(os.sched_getaffinity(0)))
orc = Wav2Vec2Oracle()
t = time.perf_counter(); a_cpu = 0
for s in segs[:args.cpu_sample]:
    orc.transcribe_ids(s); a_cpu += len(s) / 16000
out["cpu_baseline"] = {"value": a_cpu / (time.perf_counter() - t), "cores": len(os.sched_getaffinity(0)),
                       "sample": f"{args.cpu_sample} segments ({a_cpu:.1f} audio-s), oracle/ torch fp32"}
print(json.dumps(out))
