"""Does a B-frame forward depend on what frames B..max-1 of the activation
buffers hold (stale data from an earlier, larger batch)?  For each B:
forward Bmax frames of junk, then B frames of the real inputs, and compare
with a clean forward of the real inputs."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from test_generator import _inputs
from paper_2512_18318_b200 import generator
from paper_2512_18318_b200.api import Context
w = generator.synthetic_weights(0)
ctx = Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
Bmax = int(sys.argv[1]) if len(sys.argv) > 1 else 32
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 1
eng = generator.LipsyncEngine(w, max_batch=Bmax, ctx=ctx, precision=prec)
real = [torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in _inputs(Bmax, 5)]
junk = [torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in _inputs(Bmax, 99)]
junk[2] = torch.randint(0, 256, junk[2].shape, dtype=torch.uint8, device="cuda")
def run(d, B):
    out = torch.empty(B, 96, 96, 3, dtype=torch.uint8, device="cuda")
    eng.forward_device(*[t.data_ptr() for t in d], out.data_ptr(), 1, B)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(int)
ref = run(real, Bmax)
bad = []
for B in range(1, Bmax):
    run(junk, Bmax)
    o = run(real, B)
    e = np.abs(o - ref[:B]).max()
    if e > 2:
        frames = [int(i) for i in np.flatnonzero(np.abs(o - ref[:B]).reshape(B, -1).max(1) > 2)]
        bad.append((B, int(e), frames[:6]))
print("prec", prec, "Bmax", Bmax, "stale-sensitive batch sizes:", bad)
