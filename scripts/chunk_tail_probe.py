"""Device-only probe: one mba_solve over the whole config-4 batch vs the same
problems in n chunks alternating over two streams (all inputs resident), to
separate kernel-tail cost from host / PCIe cost in the end-to-end path."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "src")]


def main():
    import torch
    from paper_2506_05558_b200 import solver
    from paper_2506_05558_b200.synth import make_batch
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    b = make_batch(B, n_cams=8, K=2000, seed=0, workers=len(os.sched_getaffinity(0)))
    prm = solver.LmParams(max_iters=200, precision="f64")
    whole = solver.to_device(solver.pack_synth(b))
    sol = solver.solve(whole, prm)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record(); solver.solve(whole, prm, sol); e[1].record(); torch.cuda.synchronize()
    print("1 chunk: %.1f ms" % e[0].elapsed_time(e[1]))
    del whole, sol
    for n in (4, 8, 16, 32):
        cuts = [B * i // n for i in range(n + 1)]
        dbs, sols, wss = [], [], []
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            sub = make_batch(hi - lo, n_cams=8, K=2000, seed=0, first=lo)
            d = solver.to_device(solver.pack_synth(sub))
            dbs.append(d)
            sols.append(solver.Solution(d, prm.max_iters))
            wss.append(torch.empty(max(solver.workspace_bytes(d, prm), 16), dtype=torch.uint8, device="cuda"))
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        torch.cuda.synchronize()
        for rep in range(2):
            cur = torch.cuda.current_stream()
            e[0].record(cur)
            for i, (d, s, w) in enumerate(zip(dbs, sols, wss)):
                st = streams[i % 2]
                st.wait_event(e[0])
                with torch.cuda.stream(st):
                    solver.solve(d, prm, s, ws=w)
            for st in streams:
                cur.wait_stream(st)
            e[1].record(cur)
            torch.cuda.synchronize()
        print("%d chunks on 2 streams: %.1f ms" % (n, e[0].elapsed_time(e[1])))
        del dbs, sols, wss
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
