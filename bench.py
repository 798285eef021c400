"""Benchmark: queries/sec at recall@100 of the B200 HiPANNS hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {gmpgr,reference}]
                    [--config cfg3|cfg2|cfg1|small]

Workload (default cfg3 = BASELINE configs[2], the config the metric is quoted on):
10M items, 128-d embeddings, degree-48 graph (m=24), 3-relation MLP (64, 64),
top-100, SearchParams(k=100, k_parallel=8, hops=3, ef=200) (reference defaults,
evalharness.py:84-87), a 65,536-query batch per GPU (weak scaling: every rank holds a
replica of the index and searches its own query batch; no data-path collective).

Graph: the reference's own construction algorithm (GraphIndex.build(m=24,
ef_construction=64, seed=0), native exact parallel build, cached on the box's local
disk); the line's `own_graph` block repeats the search on this repo's bulk GPU graph
producer over the same items (--graph gpu makes that the headline instead).

A step = one batched C-HiPANNS over the per-GPU query batch = ONE launch of
hipanns_duo_kernel (tcgen05 scoring + exact refinement fused).  `value` uses device-resident
inputs, CUDA events on the launching stream, max over ranks.  `e2e` goes through the
public host API (host buffers, H2D of users + D2H of ids/scores/stats inside the
timed region).  `--impl reference` times the reference algorithm's CPU restatement
(oracle/c, all host threads) on a bounded query sample of the same workload.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PARAMS = dict(k=100, k_parallel=8, hops=3, ef=200)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# stdout carries exactly one JSON line: everything else the process (NCCL banners, library
# prints) writes to file descriptor 1 is sent to stderr, the line goes to the saved stdout
_JSON_OUT = None


def _isolate_stdout():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def emit(line: dict):
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        if self.gpu < 0:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r.split(",") for r in (self.out or "").strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][2]),
                "reasons": reasons, "samples": len(rows)}


def algorithmic_bytes(evals, rows, nbrs, d_h, k, bytes_per_elem=4):
    """B_q = 4*NbrIds + 4*Rows + s_e*d_h*E + 8k, summed over queries."""
    return float(4 * nbrs.sum() + 4 * rows.sum() + bytes_per_elem * d_h * evals.sum()
                 + 8 * k * len(evals))


def flops_per_eval(model):
    dims = [l[0].shape[0] for l in model.metric.layers]
    d_h = model.d_h
    z = dims[-1]
    f = d_h * dims[0]  # item half of layer 0 (user half hoisted per query)
    prev = dims[0]
    for o in dims[1:]:
        f += prev * o
        prev = o
    return 2 * (f + z)


def dist_setup(n_gpus):
    import torch

    if n_gpus > 1 or int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist

        rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", str(rank)))
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if os.environ.get("NCCL_DEBUG"):  # NCCL logs go to stderr: stdout is the one JSON line
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return dist, rank, dist.get_world_size(), local
    torch.cuda.set_device(0)
    return None, 0, 1, 0


def cpu_search(wl, queries, nthreads=None, params=None):
    """The reference algorithm's C restatement (oracle/c) on the host cores."""
    from oracle import oracle_c

    ids, levels, layers, entry = wl.index.graph_view()
    m = wl.model.metric
    t0 = time.perf_counter()
    r = oracle_c.search(layers, entry, ids, m.layers, m.attention, m.activation == "relu",
                        wl.items_host, queries, **(params or PARAMS), nthreads=nthreads)
    return r, time.perf_counter() - t0


def cpu_probe(wl, threads):
    """Throughput probe (2 rounds, the first absorbs per-thread visited-array setup)."""
    probe = wl.users[: max(64, 8 * threads)]
    cpu_search(wl, probe[: 2 * threads], threads)
    _, t = cpu_search(wl, probe, threads)
    return len(probe) / t


def host_threads() -> int:
    """Every host core this process may run on (torchrun sets OMP_NUM_THREADS=1, which
    must not throttle the CPU baseline)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(wl, target_s=15.0):
    threads = host_threads()
    qps = cpu_probe(wl, threads)
    n = int(min(len(wl.users), max(64, qps * target_s)))
    r, t = cpu_search(wl, wl.users[:n], threads)
    return r, n, t, threads


REF_PKG = os.path.join(ROOT, "baseline", "_ref")  # pip-installed /root/reference (nann), if present
_STOCK = {}


def _stock_one(q):
    from nann import SearchParams as RefParams, c_hipanns as ref_c_hipanns, model_scorer as ref_scorer

    g = _STOCK
    t0 = time.perf_counter()
    r = ref_c_hipanns(g["index"], ref_scorer(g["model"], g["users"][q], g["items"]), RefParams(**g["params"]))
    dt = time.perf_counter() - t0
    ids = np.full(g["params"]["k"], -1, np.int64)
    sc = np.full(g["params"]["k"], np.nan)
    for j, (i, v) in enumerate(r.items):
        ids[j], sc[j] = i, v
    return q, ids, sc, int(r.stats.metric_evaluations), dt


def stock_reference(wl, queries, params, processes=1, budget_s=None):
    """The UNMODIFIED reference package (nann, pip-installed from /root/reference into
    baseline/_ref) searching this workload: nann.GraphIndex.load of this index's NANN-IDX
    file, nann.create_model(d, d, Z, (64, 64), seed=1) (the same weights), model_scorer over
    the same item embeddings, nann.c_hipanns with the same SearchParams -- in `processes`
    forked processes.  With budget_s, queries are taken in order until the budget is spent.
    Returns (ids, scores, evals, n_done, seconds) or None when nann is not installed."""
    if not os.path.isdir(os.path.join(REF_PKG, "nann")):
        return None
    import multiprocessing as mp

    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    from nann import GraphIndex as RefIndex, create_model as ref_create_model

    cache = os.environ.get("GMPGR_CACHE", "/tmp/gmpgr_cache")
    os.makedirs(cache, exist_ok=True)
    from paper_2502_11490_b200 import workload as W

    path = os.path.join(cache, f"{wl.name}_{W.graph_digest(wl.index)[:16]}.nannidx")
    if not os.path.exists(path):
        wl.index.save(path + ".tmp")
        os.replace(path + ".tmp", path)
    d = wl.model.d_h
    _STOCK.update(index=RefIndex.load(path),
                  model=ref_create_model(d_x=d, d_h=d, z_dim=wl.model.z_dim, hidden=(64, 64), seed=1),
                  users=wl.users, items=wl.items_host, params=dict(params))
    queries = list(queries)
    out = []
    t0 = time.perf_counter()
    if processes <= 1:
        for q in queries:
            out.append(_stock_one(q))
            if budget_s and time.perf_counter() - t0 > budget_s:
                break
    else:
        with mp.get_context("fork").Pool(processes) as pool:
            for r in pool.imap(_stock_one, queries, chunksize=1):
                out.append(r)
                if budget_s and time.perf_counter() - t0 > budget_s:
                    pool.terminate()
                    break
    elapsed = time.perf_counter() - t0
    out.sort(key=lambda r: r[0])
    return (np.stack([r[1] for r in out]), np.stack([r[2] for r in out]),
            np.array([r[3] for r in out]), len(out), elapsed)


def run_reference(args):
    dist, rank, world, local = dist_setup(args.gpus)
    if rank != 0:
        return 0
    from paper_2502_11490_b200 import workload

    if args.config in ("cfg1", "cfg2"):
        wl = workload.make_reference(args.config, device=None)
    else:
        wl = workload.make(args.config, rank=0, device=local, host_items=True, graph=args.graph)
    log(f"[reference] workload {args.config} built in {wl.build_s:.1f}s")
    threads = host_threads()
    qps = cpu_probe(wl, threads)
    per_step = int(min(len(wl.users), max(64, qps * args.ref_step_s)))
    for w in range(args.warmup):
        cpu_search(wl, wl.users[:per_step], threads)
    t_tot = 0.0
    for s in range(args.steps):
        lo = (s * per_step) % max(1, len(wl.users) - per_step + 1)
        _, t = cpu_search(wl, wl.users[lo:lo + per_step], threads)
        t_tot += t
    qps = per_step * args.steps / t_tot
    line = {
        "impl": "reference", "metric": "queries/sec at recall@100", "value": qps,
        "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * t_tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_of(args, wl),
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "port",
                         "sample": f"{per_step} queries per step of the {args.config} batch, "
                                   f"oracle/c (C restatement of nann.c_hipanns + einsum-order "
                                   f"relevance), {threads} OpenMP threads"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    # the unmodified reference package itself (nann from baseline/_ref), all host cores as
    # processes, on the first queries of the same batch -- and the oracle port's agreement
    try:
        st = stock_reference(wl, range(len(wl.users)), PARAMS, processes=threads, budget_s=args.stock_s)
    except Exception as e:  # the arm's own measurement above stands; say why this one is missing
        st = None
        line["stock_reference"] = {"unavailable": f"{type(e).__name__}: {e}"[:300]}
    if st is not None:
        ids_s, sc_s, ev_s, n_s, t_s = st
        r_o, _ = cpu_search(wl, wl.users[:n_s], threads)
        line["stock_reference"] = {
            "value": n_s / t_s, "unit": "queries/s", "processes": threads,
            "sample": f"first {n_s} queries of the batch, nann.c_hipanns + model_scorer (the unmodified "
                      f"reference package, pip-installed into baseline/_ref), {threads} processes, {t_s:.1f}s",
            "oracle_port_vs_stock": parity_vs(ids_s, sc_s, ev_s, r_o["ids"], r_o["scores"], r_o["evals"])}
    emit(line)
    if dist:
        dist.destroy_process_group()
    return 0


def config_of(args, wl):
    N, d = wl.index._n, wl.model.d_h
    return {"mode": getattr(args, "mode", "exact"),
            "workload": f"{args.config}: {N} items, {d}-d, degree-{2 * wl.index.m} graph "
                        f"(m={wl.index.m}), Z={wl.model.z_dim} MLP(64,64), top-100, "
                        f"{len(wl.users)} queries per GPU",
            "params": dict(PARAMS), "n_items": N, "d_h": d, "queries_per_gpu": len(wl.users),
            "parallelism": f"query-parallel replicas x{args.gpus}",
            "l2": ("inputs larger than L2 (graph + embeddings >> 126 MB)" if N * d * 4 > 2 * 126e6
                   else "L2 flushed between timed launches (256 MB write); value = queries / sum "
                        "of launch times"),
            "graph": ("reference GraphIndex.build(m=16, ef_construction=64, seed=0) on the "
                      "reference's clustered_vectors/create_model inputs, native exact build "
                      "(graph digest identical to the reference's)" if args.config in ("cfg1", "cfg2")
                      else f"the reference's construction algorithm (GraphIndex.build m={wl.index.m}, "
                           f"ef_construction=64; native exact parallel build)" if getattr(args, "graph", "gpu") == "exact"
                      else "GPU producer (builder.py): reference level draws + symmetric pruned k-NN")}


def ncu_profile(kernel: str, per_launch_s: float, config: str, mode: str, graph: str = "gpu"):
    """The committed ncu --set full summary for THIS run's kernel, or None: the capture must
    name the same kernel instantiation, the same config/params/mode, and its launch duration
    must be within 25% of this run's CUDA-event launch time (ncu runs cold, serialised)."""
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_search_kernel.json")))
    except Exception:
        return None
    if (prof.get("config") != config or prof.get("params") != dict(PARAMS) or prof.get("mode") != mode
            or prof.get("graph", "gpu") != graph):
        return None
    for k in prof.get("kernels", []):
        if kernel not in k.get("kernel", ""):
            continue
        dur = float(k["gpu__time_duration.sum"].split()[0]) / 1e3
        if abs(dur - per_launch_s) <= 0.25 * per_launch_s:
            return prof, k
    return None


def reference_golden(config: str):
    path = os.path.join(ROOT, "tests", "golden", f"{config}_ref.npz")
    return np.load(path) if os.path.exists(path) else None


def parity_vs(ref_ids, ref_scores, ref_evals, ids, scores, evals):
    n = len(ref_ids)
    return {"queries": int(n),
            "ids_identical": float(np.mean([np.array_equal(ref_ids[q], ids[q]) for q in range(n)])),
            "scores_identical": float(np.mean([np.array_equal(ref_scores[q], scores[q], equal_nan=True)
                                               for q in range(n)])),
            "evals_identical": float(np.mean(np.asarray(ref_evals[:n]) == np.asarray(evals[:n])))}


def run_gmpgr(args):
    import torch

    dist, rank, world, local = dist_setup(args.gpus)
    from paper_2502_11490_b200 import _lib, workload
    from paper_2502_11490_b200.search import SearchParams, brute_force_batch

    dev = local
    want_cpu = (world == 1 and not args.no_cpu_baseline)
    if args.config in ("cfg1", "cfg2"):
        # BASELINE configs 1/2 on the reference's own inputs and (native exact) graph build
        wl = workload.make_reference(args.config, device=dev)
    else:
        wl = workload.make(args.config, rank=rank, device=dev, host_items=want_cpu, graph=args.graph)
    log(f"[rank {rank}] workload {args.config} built in {wl.build_s:.1f}s, "
        f"layers {wl.index.layer_node_counts()}")
    model, index = wl.model, wl.index
    metric = model.metric
    dm = metric.device_model(dev)
    g = index.device_graph(dev, items=wl.items)
    it = _lib.DeviceItems(wl.items, dev)
    searcher = _lib.DeviceSearcher(dev)
    Q, k, L, d_h = len(wl.users), PARAMS["k"], g.n_layers, model.d_h
    users_d = torch.from_numpy(wl.users).to(f"cuda:{dev}")
    out_ids = torch.empty((Q, k), dtype=torch.int64, device=f"cuda:{dev}")
    out_sc = torch.empty((Q, k), dtype=torch.float64, device=f"cuda:{dev}")
    out_cnt = torch.empty(Q, dtype=torch.int32, device=f"cuda:{dev}")
    out_st = torch.empty((Q, 5 + L), dtype=torch.int64, device=f"cuda:{dev}")
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    lib = _lib.lib()
    n_items, d_items = wl.items.shape
    flush = (torch.empty(64 << 20, dtype=torch.float32, device=f"cuda:{dev}")
             if n_items * d_items * 4 <= 2 * 126e6 else None)

    def measure(params: dict, steps: int, warmup: int, clocks: bool = False, graph=None):
        """Device-timed search launches (CUDA events on the launching stream, max over ranks)."""
        pc = SearchParams(**params, mode=args.mode, band_rel=args.band_rel, band_abs=args.band_abs)._c()
        gh = (graph or g).h

        def step():
            _lib.check(lib.gr_search_async(searcher.h, gh, dm.h, it.h, users_d.data_ptr(), Q,
                                           ctypes.byref(pc), out_ids.data_ptr(), out_sc.data_ptr(),
                                           out_cnt.data_ptr(), out_st.data_ptr(), sp))

        for _ in range(warmup):
            step()
        _lib.check(lib.gr_searcher_status(searcher.h, sp))
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        launches0 = searcher.launches
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        marks = []
        with ClockSampler(dev if clocks else -1) as clk:
            ev0.record(stream)
            for _ in range(steps):
                if flush is not None:  # working set fits in L2: evict it between launches
                    flush.add_(1)
                e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e_a.record(stream)
                step()
                e_b.record(stream)
                marks.append((e_a, e_b))
            ev1.record(stream)
            torch.cuda.synchronize(dev)
        # a tensor-core band violation anywhere in the timed launches fails the run loudly
        _lib.check(lib.gr_searcher_status(searcher.h, sp))
        launch_s = [a.elapsed_time(b) / 1000.0 for a, b in marks]
        elapsed = sum(launch_s) if flush is not None else ev0.elapsed_time(ev1) / 1000.0
        per_launch = float(np.mean(launch_s))
        if dist:
            t = torch.tensor([elapsed], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            elapsed = float(t.item())
        st = out_st.cpu().numpy()
        return dict(elapsed=elapsed, per_launch=per_launch, launches=searcher.launches - launches0,
                    evals=st[:, 0], rows=st[:, 3], nbrs=st[:, 4], clocks=clk.summary() if clocks else None,
                    ids=out_ids.cpu().numpy(), scores=out_sc.cpu().numpy())

    T0 = time.perf_counter()
    log(f"[rank {rank}] timed search")
    main_m = measure(dict(PARAMS), args.steps, args.warmup, clocks=True)
    elapsed, per_launch = main_m["elapsed"], main_m["per_launch"]
    total_q = Q * args.steps * world
    value = total_q / elapsed
    evals, rows, nbrs = main_m["evals"], main_m["rows"], main_m["nbrs"]
    dev_ids, dev_scores = main_m["ids"], main_m["scores"]

    # ---- per-query work counters of the last step -> algorithmic bytes/flops per launch
    bytes_launch = algorithmic_bytes(evals, rows, nbrs, d_h, k)
    c0 = searcher.counters()
    exact_frac = 1.0
    if args.mode == "tc":
        exact_frac = c0["exact_rescored"] / max(1, c0["tensor_scored"])
    # CUDA-core exact-fp32 work per launch: every evaluation (exact) or the re-scored band (tc)
    flops_launch = float(evals.sum()) * flops_per_eval(model) * exact_frac
    pk = peaks()
    achieved_gbs = bytes_launch / per_launch / 1e9
    sm_mhz = pk.get("sm_max_mhz", 1965.0)
    fp32_peak = 148 * 128 * sm_mhz * 1e6 / 1e12  # separate fmul/fadd issue, TFLOP/s
    kname = ("hipanns_mq_kernel" if os.environ.get("GMPGR_KERNEL") == "mq" else "hipanns_duo_kernel") \
        if d_h in (64, 128) else "hipanns_search_kernel"
    prof = ncu_profile(kname, per_launch, args.config, args.mode,
                       "reference" if args.config in ("cfg1", "cfg2") else args.graph)
    traffic = tensor_ncu = None
    if prof:
        kp_ = prof[1]
        traffic = (float(kp_["dram__bytes_read.sum"].split()[0]) + float(kp_["dram__bytes_write.sum"].split()[0])) * 1e9
        tensor_ncu = float(kp_["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"].split()[0]) / 100
    roofline = {"bound": "hbm", "achieved": achieved_gbs, "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": achieved_gbs / pk["hbm_gbs"],
                "traffic": traffic,
                "dram_frac": None if traffic is None else traffic / per_launch / 1e9 / pk["hbm_gbs"],
                "algorithmic_bytes_per_launch": bytes_launch,
                "peak_source": "MEASURED_PEAKS.json" if "_fallback" not in pk else "fallback",
                "kernel": kname,
                "traffic_source": ("profiles/ncu_search_kernel.json (ncu --set full of this config, "
                                   "params and mode; dram__bytes_read.sum + dram__bytes_write.sum "
                                   "per launch)") if prof else
                                  "null: no ncu capture of this exact kernel/config/params/mode",
                "fp32_issue": {"achieved_tflops": flops_launch / per_launch / 1e12,
                               "peak_tflops": fp32_peak,
                               "frac": flops_launch / per_launch / 1e12 / fp32_peak,
                               "note": "exact-fp32 scoring = separately rounded FMUL+FADD "
                                       "(numpy einsum order); in tc mode only the re-scored "
                                       "band runs on CUDA cores"}}

    log(f"[rank {rank}] e2e ({time.perf_counter() - T0:.0f}s)")
    # ---- e2e through the public API with host buffers (H2D users, D2H results)
    pin_users = torch.from_numpy(wl.users).pin_memory()
    h_ids = torch.empty((Q, k), dtype=torch.int64).pin_memory()
    h_sc = torch.empty((Q, k), dtype=torch.float64).pin_memory()
    h_cnt = torch.empty(Q, dtype=torch.int32).pin_memory()
    h_st = torch.empty((Q, 5 + L), dtype=torch.int64).pin_memory()
    pc_main = SearchParams(**PARAMS, mode=args.mode, band_rel=args.band_rel, band_abs=args.band_abs)._c()

    def e2e_step():
        _lib.check(lib.gr_search(searcher.h, g.h, dm.h, it.h, pin_users.data_ptr(), Q,
                                 ctypes.byref(pc_main), h_ids.data_ptr(), h_sc.data_ptr(),
                                 h_cnt.data_ptr(), h_st.data_ptr(), 0, sp))

    e2e_step()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_t = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_t], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    h2d = Q * d_h * 4
    d2h = Q * k * 16 + Q * 4 + Q * (5 + L) * 8
    assert np.array_equal(h_ids.numpy(), dev_ids), "host-API results differ from the device-timed run"

    log(f"[rank {rank}] recall ({time.perf_counter() - T0:.0f}s)")
    # ---- recall@100 vs exact brute force (GPU, all items) on a query subset
    nrec = min(Q, args.recall_queries)
    gt_ids, _ = brute_force_batch(metric, wl.users[:nrec], wl.items, 100, device=dev)

    def recall_of(ids):
        return float(np.mean([len(set(ids[q]) & set(gt_ids[q])) / 100.0 for q in range(nrec)]))

    line = {
        "metric": "queries/sec at recall@100", "value": value, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * elapsed / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_of(args, wl),
        "recall_at_100": recall_of(dev_ids), "recall_queries": nrec,
        "mean_evals_per_query": float(evals.mean()),
        "roofline": roofline,
        "e2e": {"value": total_q / e2e_t, "unit": "queries/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": int(main_m["launches"]),
        "clocks": main_m["clocks"],
        "scoring_mode": args.mode,
    }
    if args.mode == "tc":
        frac = c0["exact_rescored"] / max(1, c0["tensor_scored"])
        line["tc_scoring"] = dict(c0, exact_rescored_frac=frac)
        # issued tcgen05 work: 3 bf16 MMAs (hi.hi, hi.lo, lo.hi) x 2 x (d_h*64 + 64*64) per evaluation
        tflop = 3 * 2 * (d_h * 64 + 64 * 64) * float(evals.sum()) / per_launch / 1e12
        pk_t = pk.get("bf16_tflops_sustained", 1408.5)
        roofline["tensor_pipe"] = {
            "frac": tensor_ncu,
            "source": "ncu sm__pipe_tensor_cycles_active (profiles/ncu_search_kernel.json)" if prof
                      else "null: no ncu capture of this exact kernel/config/params/mode",
            "issued_tflops": tflop, "issued_frac_of_bf16_peak": tflop / pk_t,
            "peak_tflops": pk_t, "peak_source": "MEASURED_PEAKS.json bf16 sustained"}
    gold = reference_golden(args.config)
    if gold is not None and rank == 0:
        # the reference's own c_hipanns / brute_force results on these exact inputs
        # (tests/golden/make_cfg_golden.py ran nann in the build container)
        import paper_2502_11490_b200.workload as W

        pi = next((i for i in range(4) if f"p{i}/params" in gold.files and
                   list(gold[f"p{i}/params"]) == [PARAMS["k"], PARAMS["k_parallel"], PARAMS["hops"], PARAMS["ef"]]),
                  None)
        rp = {"source": f"tests/golden/{args.config}_ref.npz (nann.c_hipanns + brute_force)",
              "graph_identical_to_reference_build": W.graph_digest(index) == str(gold["graph_sha256"])}
        if pi is not None:
            n = gold[f"p{pi}/res_ids"].shape[0]
            rp.update(parity_vs(gold[f"p{pi}/res_ids"], gold[f"p{pi}/res_scores"], gold[f"p{pi}/res_evals"],
                                dev_ids[:n], dev_scores[:n], evals[:n]))
            ng = min(n, gold["gt100"].shape[0])
            rp["recall_at_100_vs_reference_gt"] = float(np.mean(
                [len(set(dev_ids[q]) & set(gold["gt100"][q])) / 100.0 for q in range(ng)]))
            rp["reference_recall_at_100"] = float(gold[f"p{pi}/recall100"])
        line["reference_parity"] = rp
    log(f"[rank {rank}] operating points ({time.perf_counter() - T0:.0f}s)")
    # ---- further operating points of the same workload (higher recall budgets)
    if args.operating_points and rank == 0 or (args.operating_points and dist):
        ops = []
        for kp, hops in ((32, 10),):
            if (kp, hops) == (PARAMS["k_parallel"], PARAMS["hops"]):
                continue
            prm = dict(PARAMS, k_parallel=kp, hops=hops)
            m = measure(prm, 2, 1)
            b = algorithmic_bytes(m["evals"], m["rows"], m["nbrs"], d_h, k)
            op = {"params": prm, "value": Q * 2 * world / m["elapsed"], "unit": "queries/s",
                  "ms_per_step": 1000 * m["elapsed"] / 2, "recall_at_100": recall_of(m["ids"]),
                  "mean_evals_per_query": float(m["evals"].mean()),
                  "roofline_frac": b / m["per_launch"] / 1e9 / pk["hbm_gbs"]}
            if want_cpu and rank == 0 and wl.items_host is not None:
                nq = min(Q, 48)
                r, _ = cpu_search(wl, wl.users[:nq], host_threads(), params=prm)
                op["cpu_reference_check"] = parity_vs(r["ids"], r["scores"], r["evals"], m["ids"][:nq],
                                                      m["scores"][:nq], m["evals"][:nq])
            ops.append(op)
        line["operating_points"] = ops
    log(f"[rank {rank}] own graph ({time.perf_counter() - T0:.0f}s)")
    line["resident_units"] = searcher.counters().get("resident_units")
    # ---- the same queries on this repo's own bulk GPU graph producer (builder.py): a second
    # graph of the same items (the exact-graph line above is the reference-faithful headline)
    if args.graph == "exact" and args.own_graph and args.config not in ("cfg1", "cfg2"):
        t0 = time.perf_counter()
        from paper_2502_11490_b200.index import GraphIndex

        gidx = GraphIndex.build(wl.items, m=index.m, seed=0, device=torch.device("cuda", dev), method="gpu")
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()
        g2 = gidx.device_graph(dev, items=wl.items)
        build2 = time.perf_counter() - t0
        own = {"graph": "GPU producer (builder.py): reference level draws + symmetric pruned k-NN",
               "build_s": build2, "points": []}
        for prm, steps in ((dict(PARAMS), 3), (dict(PARAMS, k_parallel=32, hops=10), 2)):
            if not args.operating_points and prm != dict(PARAMS):
                continue
            m = measure(prm, steps, 1, graph=g2)
            b = algorithmic_bytes(m["evals"], m["rows"], m["nbrs"], d_h, k)
            own["points"].append({"params": prm, "value": Q * steps * world / m["elapsed"], "unit": "queries/s",
                                  "ms_per_step": 1000 * m["elapsed"] / steps, "recall_at_100": recall_of(m["ids"]),
                                  "mean_evals_per_query": float(m["evals"].mean()),
                                  "roofline_frac": b / m["per_launch"] / 1e9 / pk["hbm_gbs"]})
        line["own_graph"] = own
        del g2, gidx
    log(f"[rank {rank}] cpu baseline + stock reference ({time.perf_counter() - T0:.0f}s)")
    if want_cpu and rank == 0:
        r, n, t, threads = cpu_baseline(wl, target_s=args.cpu_s)
        line["cpu_baseline"] = {"value": n / t, "unit": "queries/s", "cores": threads,
                                "kind": "port",
                                "sample": f"first {n} queries of the batch, oracle/c (C "
                                          f"restatement of nann.c_hipanns + einsum-order "
                                          f"relevance), {threads} threads, {t:.1f}s"}
        line["cpu_reference_check"] = parity_vs(r["ids"], r["scores"], r["evals"], dev_ids[:n],
                                                dev_scores[:n], evals[:n])
        line["ids_identical_to_cpu_reference"] = line["cpu_reference_check"]["ids_identical"]
        # the unmodified reference package (nann, baseline/_ref) on the first queries
        nq = min(Q, args.stock_queries)
        try:
            st = stock_reference(wl, range(nq), PARAMS, processes=1) if nq else None
        except Exception as e:
            st = None
            line["stock_reference_check"] = {"unavailable": f"{type(e).__name__}: {e}"[:300]}
        if st is not None:
            ids_s, sc_s, ev_s, n_s, t_s = st
            line["stock_reference_check"] = dict(
                parity_vs(ids_s, sc_s, ev_s, dev_ids[:n_s], dev_scores[:n_s], evals[:n_s]),
                source="nann.c_hipanns + model_scorer, unmodified reference package (baseline/_ref)",
                seconds_per_query_1_process=t_s / max(1, n_s))
    if rank == 0:
        emit(line)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_sharded(args):
    """BASELINE config 4: catalog sharded over ranks (12.5M items per GPU: 100M at N=8),
    every rank searches ALL queries on its shard, per-shard top-k lists meet through an
    NCCL all-gather and the device merge (gr_merge_topk).  value = queries / step time."""
    import torch

    dist, rank, world, local = dist_setup(args.gpus)
    from paper_2502_11490_b200 import workload
    from paper_2502_11490_b200.distributed import ShardedSearcher, gather_lists, merge_packed
    from paper_2502_11490_b200.search import SearchParams, brute_force_batch

    wl = workload.make_shard(rank, world, shard_n=args.shard_n, n_queries=args.queries,
                             device=local)
    log(f"[rank {rank}] shard built in {wl.build_s:.1f}s, layers {wl.index.layer_node_counts()}")
    ss = ShardedSearcher(wl.index, wl.model, wl.items, device=local)
    users_d = torch.from_numpy(wl.users).to(f"cuda:{local}")
    params = SearchParams(**PARAMS, mode=args.mode)
    for _ in range(args.warmup):
        ss.search(users_d, params)
    torch.cuda.synchronize(local)
    if dist:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            out = ss.search(users_d, params)
        ev1.record()
        torch.cuda.synchronize(local)
    elapsed = ev0.elapsed_time(ev1) / 1000.0
    if dist:
        t = torch.tensor([elapsed], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    Q = len(wl.users)
    # recall@100 vs the global exact top-100 (per-shard exact top-100, same gather + merge)
    nrec = min(Q, args.recall_queries)
    gi, gsc = brute_force_batch(wl.model, wl.users[:nrec], wl.items, 100, device=local)
    gi = torch.from_numpy(gi + rank * args.shard_n).to(f"cuda:{local}")
    gsc = torch.from_numpy(gsc).to(f"cuda:{local}")
    gt, _, _ = merge_packed(gather_lists(gi, gsc), 100)
    got = out[0][:nrec].cpu().numpy()
    gt = gt.cpu().numpy()
    recall = float(np.mean([len(set(got[q]) & set(gt[q])) / 100.0 for q in range(nrec)]))
    line = {
        "metric": "queries/sec at recall@100", "value": Q * args.steps / elapsed, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * elapsed / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"cfg4: {args.shard_n * world} items sharded {args.shard_n}/GPU, "
                               f"128-d, degree-48 graphs, Z=3, top-100, {Q} queries, all-gather merge",
                   "params": dict(PARAMS), "mode": args.mode,
                   "parallelism": f"catalog shards x{world} + NCCL all-gather"},
        "recall_at_100": recall, "recall_queries": nrec, "clocks": clk.summary(),
        "scoring_mode": args.mode,
    }
    if rank == 0:
        emit(line)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    _isolate_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gmpgr", choices=["gmpgr", "reference"])
    ap.add_argument("--config", default="cfg3", choices=["cfg1", "cfg2", "cfg3", "cfg4", "small"])
    ap.add_argument("--shard-n", type=int, default=12_500_000, help="cfg4 items per GPU")
    ap.add_argument("--queries", type=int, default=65_536, help="cfg4 query batch")
    ap.add_argument("--recall-queries", type=int, default=256)
    ap.add_argument("--cpu-s", type=float, default=15.0)
    ap.add_argument("--ref-step-s", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stock-queries", type=int, default=16,
                    help="queries checked against the unmodified reference package (baseline/_ref)")
    ap.add_argument("--stock-s", type=float, default=20.0,
                    help="--impl reference: seconds of the unmodified reference package's timing")
    ap.add_argument("--band-rel", type=float, default=0.0,
                    help="tc-mode refinement band (relative part); <= 0: library default")
    ap.add_argument("--band-abs", type=float, default=0.0)
    ap.add_argument("--graph", default="exact", choices=["gpu", "exact"],
                    help="cfg3 graph: exact (default) = the reference's own construction algorithm "
                         "(GraphIndex.build, native exact parallel build: ~3.5 min at 10M items on "
                         "16 host cores, cached under GMPGR_CACHE for later runs on the box); gpu = "
                         "the bulk GPU producer (builder.py, ~20 s)")
    ap.add_argument("--no-own-graph", dest="own_graph", action="store_false",
                    help="skip the extra record on the GPU-producer graph (exact-graph runs)")
    ap.add_argument("--no-operating-points", dest="operating_points", action="store_false",
                    help="skip the extra kp=32/hops=10 (high-recall) operating point")
    ap.add_argument("--k-parallel", type=int, default=PARAMS["k_parallel"],
                    help="search budget override (default: the reference's evalharness defaults)")
    ap.add_argument("--hops", type=int, default=PARAMS["hops"])
    ap.add_argument("--ef", type=int, default=PARAMS["ef"])
    ap.add_argument("--mode", default="tc", choices=["exact", "tc"],
                    help="exact: CUDA-core exact-fp32 scoring; tc: tcgen05 split-bf16 scoring "
                         "with exact re-scoring of every near-threshold item")
    args = ap.parse_args()
    PARAMS.update(k_parallel=args.k_parallel, hops=args.hops, ef=args.ef)
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "cfg4":
        return run_sharded(args)
    return run_gmpgr(args)


if __name__ == "__main__":
    sys.exit(main())
