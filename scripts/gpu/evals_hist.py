"""Per-iteration trial evaluations on config 4 (how many cost passes the LM
loop runs): histogram of evals over executed iterations."""
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [REPO, os.path.join(REPO, "src")]
import numpy as np
import torch
from paper_2506_05558_b200 import solver
from paper_2506_05558_b200.synth import make_batch
b = make_batch(4096, n_cams=8, K=2000, seed=0)
db = solver.to_device(solver.pack_synth(b))
sol = solver.solve(db, solver.LmParams(max_iters=200))
torch.cuda.synchronize()
it = sol.n_iters.cpu().numpy()
ev = sol.evals.cpu().numpy().reshape(len(it), -1)
acc = sol.accepted.cpu().numpy().reshape(len(it), -1)
mask = np.arange(ev.shape[1])[None, :] < it[:, None]
e = ev[mask]
print("iters/problem", it.mean(), "evals/iter", e.mean(), "hist", np.bincount(e, minlength=6).tolist(),
      "accepted frac", acc[mask].mean())
