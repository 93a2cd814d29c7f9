import sys, json, torch
sys.path.insert(0, '.')
import ttsynth
from paper_2601_08217_b200 import Channel
dev = torch.device('cuda', 0)
res = {}
base = ttsynth.get('c4').scaled(ues=64)   # 128 channels: c4 at 8 GPUs per rank
for n, reps in ((61440, 10), (614400, 1)):
    w = base.scaled(n_per_call=n, calls=reps * 40)
    C = w.C
    K = (reps * 40 * n) // w.S + 3
    P = max(2, (4 * 126 * 2**20) // (C * n * 8) + 1)
    xs = [ttsynth.iq(w, 0, C, i, backend='torch', device=dev) for i in range(P)]
    y = torch.empty_like(xs[0])
    ch = Channel(ttsynth.delays(w), w.S, seed=1, snapshot_capacity=K, device=dev)
    ch.load_snapshots(ttsynth.snapshots(w, 0, C, K, backend='torch', device=dev), 0)
    for i in range(reps * 3):
        ch.apply(xs[i % P], out=y, noise_sigma=w.sigma)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps * 30):
        ch.apply(xs[i % P], out=y, noise_sigma=w.sigma)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (reps * 30)
    res[n] = {"ms_per_call": ms, "us_per_61440": ms * 1e3 * 61440 / n, "pool": P}
    ch.close()
    del xs
    torch.cuda.empty_cache()
print(json.dumps(res))
