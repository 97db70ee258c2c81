"""C4 fwd+bwd step time and iterations for PCG vs FGMRES(m):  python tools/fgmres_sweep.py m1 m2 ...
(m = 0 -> PCG).  MPDE_GM_REORTH=0 in the environment selects one Gram-Schmidt pass."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2502_18377_b200 import mpde  # noqa: E402

bt = synth.make_batch("C4")
g = synth.make_g("C4")
cfg = bt["cfg"]
dev = lambda a: torch.from_numpy(a).cuda()
c, b, om, gz = dev(bt["c"]), dev(bt["b"]), dev(bt["omega"]), dev(g)
for m in [int(x) for x in sys.argv[1:]]:
    o = mpde.mpde_default_options(krylov=1, restart=m) if m else mpde.mpde_default_options()
    times = []
    for it in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        s = mpde.Solver(cfg.shape, cfg.h, c, opts=o)
        z = s.forward(b, om)
        fi = [x["iters"] for x in s.stats_list()]
        s.backward(b, z, gz)
        e1.record()
        torch.cuda.synchronize()
        bi = [x["iters"] for x in s.stats_list()]
        s.close()
        times.append(e0.elapsed_time(e1))
    print(f"m={m} reorth={os.environ.get('MPDE_GM_REORTH', '1')} ms/step {min(times):.1f} "
          f"fwd its {sum(fi) / len(fi):.1f} (max {max(fi)}) bwd its {sum(bi) / len(bi):.1f} (max {max(bi)})",
          flush=True)
