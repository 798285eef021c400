"""Summarise an ncu report (`--set full`) and a launch-list CSV into profiles/.

    python tools/ncu_summary.py <report.ncu-rep> <launches.csv> <n_queries> <out_prefix>
                                [config k,kp,hops,ef mode [graph]]

The optional trailer records what was captured (bench.py only uses a capture's traffic /
tensor-pipe figures when config, params and mode match its own run).

Writes <out_prefix>.json (key metrics per captured kernel + dram bytes per query) and
<out_prefix>_sass_mix.txt (instruction mix / stall reasons of the top kernel).
"""

import csv
import io
import json
import subprocess
import sys
from collections import Counter

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_shared_mem", "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def ncu_csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, launches, nq, prefix = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
    rows = ncu_csv([rep, "--page", "raw"])
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        kernels.append(d)
    top = kernels[0] if kernels else {}

    def num(key):
        v, u = top.get(key, "0 ").split(" ", 1) if top.get(key) else ("0", "")
        v = float(v.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
                 "ms": 1e-3, "s": 1}.get(u.strip(), 1)
        return v * scale

    dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    # launch list: share of each kernel
    lrows = []
    with open(launches) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.reader(io.StringIO("".join(lines)))
    lh = next(rd)
    per = Counter()
    cnt = Counter()
    for r in rd:
        if r[lh.index("Metric Name")] == "gpu__time_duration.sum":
            name = r[lh.index("Kernel Name")]
            per[name] += float(r[lh.index("Metric Value")].replace(",", ""))
            cnt[name] += 1
    tot = sum(per.values()) or 1.0
    share = {k: {"launches": cnt[k], "total_ns": v, "share": v / tot} for k, v in per.items()}
    extra = {}
    if len(sys.argv) > 7:
        k, kp, hops, ef = (int(v) for v in sys.argv[6].split(","))
        extra = {"config": sys.argv[5], "params": {"k": k, "k_parallel": kp, "hops": hops, "ef": ef},
                 "mode": sys.argv[7], "graph": sys.argv[8] if len(sys.argv) > 8 else "gpu"}
    summary = {"report": rep, "n_queries": nq, **extra, "kernels": kernels,
               "dram_bytes_per_launch": dram, "dram_bytes_per_query": dram / max(1, nq),
               "launch_list": share}
    json.dump(summary, open(prefix + ".json", "w"), indent=1)
    # instruction mix + stalls of the captured kernel
    src = ncu_csv([rep, "--page", "source"])
    h = src[1]
    data = src[2:]
    ix = {k: i for i, k in enumerate(h)}

    def f(r, k):
        try:
            return float(r[ix[k]])
        except Exception:
            return 0.0

    ops, samp = Counter(), Counter()
    for r in data:
        toks = r[ix["Source"]].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        ops[op] += f(r, "Instructions Executed")
        samp[op] += f(r, "Warp Stall Sampling (All Samples)")
    ti = sum(ops.values()) or 1
    ts = sum(samp.values()) or 1
    stalls = {k: sum(f(r, k) for r in data) for k in h if k.startswith("stall_") and "Not Issued" not in k}
    with open(prefix + "_sass_mix.txt", "w") as out:
        out.write(f"instructions executed: {ti:.4g}\n")
        for op, c in ops.most_common(25):
            out.write(f"{op:10s} {100 * c / ti:5.1f}% of instructions  {100 * samp[op] / ts:5.1f}% of stall samples\n")
        out.write("\nstall reasons (samples):\n")
        for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:12]:
            out.write(f"  {k:28s} {v:10.0f}\n")
    # hottest CUDA source lines (warp-stall samples, correlated through -lineinfo)
    rows = ncu_csv([rep, "--page", "source", "--print-source", "cuda,sass"])
    cur, hdr2, agg, text, why = None, None, Counter(), {}, {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr2 = r
            continue
        if r[0] == "Function Name" or hdr2 is None or not r[0]:
            continue
        key = (cur, int(r[0]))
        text[key] = r[1].strip()
        try:
            agg[key] += float(r[4] or 0)
            c = why.setdefault(key, Counter())
            for i, name in enumerate(hdr2):
                if name.startswith("stall_") and "Not Issued" not in name and r[i]:
                    c[name] += float(r[i])
        except ValueError:
            pass
    tot = sum(agg.values()) or 1.0
    with open(prefix + "_lines.txt", "w") as out:
        out.write("share of warp-stall samples by CUDA source line (top 40) and main stall reasons\n")
        for key, v in agg.most_common(40):
            c = why.get(key, Counter())
            tw = sum(c.values()) or 1.0
            rs = ", ".join(f"{k[6:]} {100 * x / tw:.0f}%" for k, x in c.most_common(2))
            out.write(f"{100 * v / tot:5.2f}%  {key[0]}:{key[1]:<5d} {text[key][:70]:70s}  [{rs}]\n")
    print(json.dumps({k: summary[k] for k in ("dram_bytes_per_query", "launch_list")}, indent=1))


if __name__ == "__main__":
    main()
