"""BASELINE config 5 sweep: 1M items, 128-d, degree-32 graph (m=16), Z=3, top-100;
beam width (ef) x k_parallel x hops x query batch -> QPS and recall@100 (recall/QPS Pareto).

    python tools/sweep.py [out.json] [--quick]
"""

import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_11490_b200 import _lib, workload  # noqa: E402
from paper_2502_11490_b200.search import SearchParams, brute_force_batch  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "gpurun_out/sweep.json"
    quick = "--quick" in sys.argv
    torch.cuda.set_device(0)
    Qmax = 262_144
    workload.CONFIGS["cfg5"] = (1_000_000, 128, 16, 1024, 3, Qmax)
    wl = workload.make("cfg5", n_queries=Qmax)
    print(f"built in {wl.build_s:.1f}s layers {wl.index.layer_node_counts()}", flush=True)
    dm = wl.model.metric.device_model(0)
    g = wl.index.device_graph(0, items=wl.items)
    it = _lib.DeviceItems(wl.items, 0)
    s = _lib.DeviceSearcher(0)
    users = torch.from_numpy(wl.users).cuda()
    nrec = 256
    gt, _ = brute_force_batch(wl.model, wl.users[:nrec], wl.items, 100)
    lib = _lib.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    rows = []
    efs = [32, 64, 128, 256]
    kps = [(8, 3), (32, 10)] if not quick else [(8, 3)]
    batches = [1024, 4096, 16384, 65536, 262144] if not quick else [65536]
    for kp, hops in kps:
        for ef in efs:
            for Q in batches:
                pc = SearchParams(k=100, k_parallel=kp, hops=hops, ef=ef, mode="tc")._c()
                L = g.n_layers
                oi = torch.empty((Q, 100), dtype=torch.int64, device="cuda")
                osc = torch.empty((Q, 100), dtype=torch.float64, device="cuda")
                oc = torch.empty(Q, dtype=torch.int32, device="cuda")
                ost = torch.empty((Q, 5 + L), dtype=torch.int64, device="cuda")

                def run():
                    _lib.check(lib.gr_search_async(s.h, g.h, dm.h, it.h, users.data_ptr(), Q,
                                                   ctypes.byref(pc), oi.data_ptr(), osc.data_ptr(),
                                                   oc.data_ptr(), ost.data_ptr(), st))

                run()
                _lib.check(lib.gr_searcher_status(s.h, st))
                reps = max(1, min(5, int(4 * 65536 / Q)))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    run()
                e1.record()
                torch.cuda.synchronize()
                _lib.check(lib.gr_searcher_status(s.h, st))
                t = e0.elapsed_time(e1) / 1000 / reps
                ids = oi[:nrec].cpu().numpy()
                rec = float(np.mean([len(set(ids[q]) & set(gt[q])) / 100 for q in range(min(nrec, Q))]))
                ev = float(ost[:, 0].float().mean())
                row = dict(k_parallel=kp, hops=hops, ef=ef, batch=Q, qps=Q / t,
                           recall_at_100=rec, evals_per_query=ev, ms=t * 1e3)
                rows.append(row)
                print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    json.dump({"workload": "cfg5: 1M items, 128-d, m=16 (degree 32), Z=3 MLP(64,64), top-100, "
                           "tc mode (tcgen05 + exact refinement), synthetic clustered (1024)",
               "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
