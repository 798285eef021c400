"""Launch hipanns_search_kernel a few times on a synthetic workload (for ncu captures).

    python tools/profile_search.py [config] [n_queries] [launches]
"""

import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_11490_b200 import _lib, workload  # noqa: E402
from paper_2502_11490_b200.search import SearchParams  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "small"
    nq = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    kw = dict(k=100, k_parallel=8, hops=3, ef=200)
    if len(sys.argv) > 4 and sys.argv[4] != "-":
        kp, hops = (int(v) for v in sys.argv[4].split("x"))
        kw.update(k_parallel=kp, hops=hops)
    if len(sys.argv) > 5:
        kw["mode"] = sys.argv[5]
    if os.environ.get("BAND"):
        kw["band_rel"] = kw["band_abs"] = float(os.environ["BAND"])
    torch.cuda.set_device(0)
    wl = workload.make(cfg, n_queries=nq, graph=os.environ.get("GMPGR_GRAPH", "gpu"),
                       n_items=int(os.environ["GMPGR_NITEMS"]) if os.environ.get("GMPGR_NITEMS") else None)
    print(f"workload {cfg}: {wl.index._n} items, built in {wl.build_s:.1f}s", flush=True)
    dm = wl.model.metric.device_model(0)
    g = wl.index.device_graph(0, items=wl.items)
    it = _lib.DeviceItems(wl.items, 0)
    s = _lib.DeviceSearcher(0)
    Q, k, L = nq, kw["k"], g.n_layers
    users = torch.from_numpy(wl.users).cuda()
    oi = torch.empty((Q, k), dtype=torch.int64, device="cuda")
    osc = torch.empty((Q, k), dtype=torch.float64, device="cuda")
    oc = torch.empty(Q, dtype=torch.int32, device="cuda")
    ost = torch.empty((Q, 5 + L), dtype=torch.int64, device="cuda")
    pc = SearchParams(**kw)._c()
    lib = _lib.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    # ncu --profile-from-start off: only the search launches are profiled (the workload
    # builder's thousands of small kernels stay outside the capture range)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(lib.gr_search_async(s.h, g.h, dm.h, it.h, users.data_ptr(), Q, ctypes.byref(pc),
                                       oi.data_ptr(), osc.data_ptr(), oc.data_ptr(), ost.data_ptr(), st))
        _lib.check(lib.gr_searcher_status(s.h, st))
        dt = time.perf_counter() - t0
        stats = ost.cpu().numpy()
        print(f"launch {r}: {dt*1e3:.2f} ms  {Q/dt:.0f} q/s  evals/q {stats[:,0].mean():.1f} "
              f"rows/q {stats[:,3].mean():.1f} nbrs/q {stats[:,4].mean():.1f}", flush=True)
    torch.cuda.profiler.stop()
    print("counters", s.counters(), flush=True)
    free, total = torch.cuda.mem_get_info()
    print(f"device memory: {(total - free) / 1e9:.1f} GB in use of {total / 1e9:.1f} GB", flush=True)


if __name__ == "__main__":
    main()
