import sys, collections, json
sys.path.insert(0, '.')
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_2507_01021_b200.ctc import Wav2Vec2GPU
rng = np.random.default_rng(5)
segs = [rng.integers(-8000, 8000, size=int(rng.uniform(1, 8) * 16000), dtype=np.int16) for _ in range(64)]
eng = Wav2Vec2GPU(max_batch=64, max_samples=8 * 16000)
flat = np.concatenate(segs); pcm = torch.from_numpy(flat).cuda()
offs = np.cumsum([0] + [len(s) for s in segs[:-1]]).tolist()
for _ in range(3): eng.run(segs, resident=(pcm, offs))
eng.stream.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.run(segs, resident=(pcm, offs)); eng.stream.synchronize()
fam = collections.defaultdict(list)
for e in prof.events():
    if e.device_type.name == "CUDA" and e.device_time_total > 0:
        fam[e.name.split("(")[0].replace("void ", "")].append(e.device_time_total)
tot = sum(sum(v) for v in fam.values())
print("total us", round(tot,1), "audio s", sum(len(s) for s in segs)/16000)
for k, v in sorted(fam.items(), key=lambda kv: -sum(kv[1]))[:14]:
    print(f"{k[:60]:60s} n={len(v):4d} mean={sum(v)/len(v):8.1f} total={sum(v):9.1f} {100*sum(v)/tot:5.1f}%")
