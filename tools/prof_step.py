"""One C4 fwd+bwd step (batch 32) for ncu captures: python tools/prof_step.py [steps]"""
import sys, os, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
from paper_2502_18377_b200 import mpde
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
bt = synth.make_batch("C4"); g = synth.make_g("C4"); cfg = bt["cfg"]
dev = lambda a: torch.from_numpy(a).cuda()
c, b, om, gz = dev(bt["c"]), dev(bt["b"]), dev(bt["omega"]), dev(g)
for _ in range(steps):
    s = mpde.Solver(cfg.shape, cfg.h, c)
    z = s.forward(b, om)
    s.backward(b, z, gz)
    torch.cuda.synchronize()
    s.close()
print("ok", s.stats_list()[0])
