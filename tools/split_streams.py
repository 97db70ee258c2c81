"""Experiment: one B=32 C4 solve vs two B=16 halves on two streams from two host threads
(overlap of one half's latency-bound coarse levels / launch gaps with the other's level-0
kernels).  Dev tool (GPU)."""
import os, sys, threading, time, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
from paper_2502_18377_b200 import mpde
bt = synth.make_batch("C4"); g = synth.make_g("C4"); cfg = bt["cfg"]
dev = lambda a: torch.from_numpy(a).cuda()
c, b, om, gz = dev(bt["c"]), dev(bt["b"]), dev(bt["omega"]), dev(g)

def run(lo, hi, stream, reps, out):
    with torch.cuda.stream(stream):
        for _ in range(reps):
            s = mpde.Solver(cfg.shape, cfg.h, c[lo:hi].contiguous(), stream=stream)
            z = s.forward(b[lo:hi].contiguous(), om[lo:hi].contiguous(), stream=stream)
            s.backward(b[lo:hi].contiguous(), z, gz[lo:hi].contiguous(), stream=stream)
            stream.synchronize()
            s.close()
    out.append(1)

for split in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(split)]
    n = 32 // split
    # warm-up sequentially (graph capture uses one private stream)
    for k in range(split):
        run(k * n, (k + 1) * n, streams[k], 1, [])
    torch.cuda.synchronize()
    reps = 4
    t0 = time.perf_counter()
    ths = [threading.Thread(target=run, args=(k * n, (k + 1) * n, streams[k], reps, [])) for k in range(split)]
    [t.start() for t in ths]; [t.join() for t in ths]
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"split {split}: {1e3 * dt:.1f} ms per 32-PDE fwd+bwd -> {32 / dt:.1f} solves/s", flush=True)
