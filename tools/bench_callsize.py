import sys, json, torch
sys.path.insert(0, '.')
import ttsynth
from paper_2601_08217_b200 import Channel
dev = torch.device('cuda', 0)
res = {}
for n, reps in ((30720, 10), (307200, 1), (61440, 5), (15360, 20)):
    w = ttsynth.get('c3').scaled(n_per_call=n, calls=reps * 30)
    C = w.C
    K = (reps * 30 * n) // w.S + 3
    xs = [ttsynth.iq(w, 0, C, i, backend='torch', device=dev) for i in range(4)]
    y = torch.empty_like(xs[0])
    ch = Channel(ttsynth.delays(w), w.S, seed=1, snapshot_capacity=K, device=dev)
    ch.load_snapshots(ttsynth.snapshots(w, 0, C, K, backend='torch', device=dev), 0)
    for i in range(reps * 3):
        ch.apply(xs[i % 4], out=y, noise_sigma=w.sigma)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps * 20):
        ch.apply(xs[i % 4], out=y, noise_sigma=w.sigma)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (reps * 20)
    res[n] = {"ms_per_call": ms, "us_per_30720": ms * 1e3 * 30720 / n}
    ch.close()
print(json.dumps(res))
