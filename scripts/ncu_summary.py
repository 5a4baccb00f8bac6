"""Summarise a round's ncu evidence (scripts/profile_round.sh) into profiles/:
  <R>_ncu_launches.md   per-kernel share of the bench command's launch list
  <R>_ncu_full.md       one --set full capture per hot kernel (duration, DRAM bytes, pipes)
  ncu_traffic.json      DRAM bytes per launch per kernel (read by bench.py for roofline.traffic)
usage: python scripts/ncu_summary.py r01 [gpurun_out]"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
D = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def short(name):
    name = name.split("(")[0]
    return name.replace("void ", "").strip()


def launches():
    path = os.path.join(D, "launches_%s.csv" % R)
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}.get(unit, 1)
        a = agg[short(r["Kernel Name"])]
        a[0] += 1
        a[1] += ns
    tot = sum(a[1] for a in agg.values())
    out = ["# ncu launch list — `python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline` (%s)" % R, "",
           "`ncu --metrics gpu__time_duration.sum --clock-control none` over the whole command (warm-up, timed",
           "steps, instrumented chunk; kernels replayed from the CUDA graph are listed per node). Per-launch",
           "times are serialised and cold-cache, so compare SHARES with bench.py's per_kind breakdown.", "",
           "| kernel | launches | total ms | share | avg us |", "|---|---|---|---|---|"]
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append("| %s | %d | %.1f | %.1f %% | %.1f |" % (k, n, ns / 1e6, 100 * ns / tot, ns / n / 1e3))
    open(os.path.join(PROF, "%s_ncu_launches.md" % R), "w").write("\n".join(out) + "\n")
    return agg


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__cycles_active.avg",
           "gpc__cycles_elapsed.max", "smsp__cycles_active.avg.per_second"]
SHAPES = {"gemm": "QKV-shape GEMM 10530x15360x5120 (bf16 epilogue)", "fmha": "self-attn L=10530, 40 heads, hd 128",
          "cross": "cross-attn Lq=10530, Lk=37, 40 heads", "conv": "VAE conv 96->96 3x3x3, 28x416x720 (fp32 out)",
          "xpb": "folded cross-attn output GEMM 10530x5120x1600 (fp32 residual + gate)",
          "norm": "norm+AdaLN 10530x5120 f32 -> bf16",
          "xs": "folded cross-attn logits GEMM 10530x1792x5120 + per-head softmax epilogue (bf16 P)"}


def full():
    res = {}
    for w in ("gemm", "fmha", "xpb", "xs", "cross", "conv", "norm"):
        rep = os.path.join(D, "full_%s_%s.ncu-rep" % (R, w))
        if not os.path.exists(rep):
            continue
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        h, units, v = rows[0], rows[1], rows[2]
        d = {k: (val, u) for k, u, val in zip(h, units, v)}
        res[w] = {"kernel": short(d["Kernel Name"][0])}
        for m in METRICS:
            if m in d:
                val, u = d[m]
                try:
                    res[w][m] = (float(val.replace(",", "")), u)
                except ValueError:
                    pass
    return res


def to_bytes(x):
    v, u = x
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def to_us(x):
    v, u = x
    return v * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}.get(u, 1)


def main():
    os.makedirs(PROF, exist_ok=True)
    agg = launches() if os.path.exists(os.path.join(D, "launches_%s.csv" % R)) else {}
    res = full()
    out = ["# ncu --set full, one launch per hot kernel (%s) — `scripts/profile_round.sh`" % R, "",
           "`ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 1 -c 1` on",
           "`scripts/profile_kernels.py <kernel>` (14B shapes), after the same command exited 0 without ncu.", "",
           "| kernel | shape | us | DRAM read MB | DRAM write MB | tensor pipe % | SM thr % | DRAM thr % | XU % | issue % | regs |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for w, d in res.items():
        g = lambda m: d.get(m, (float("nan"), ""))[0]  # noqa: E731
        rd, wr = to_bytes(d["dram__bytes_read.sum"]), to_bytes(d["dram__bytes_write.sum"])
        us = to_us(d["gpu__time_duration.sum"])
        traffic[w] = {"kernel": d["kernel"], "shape": SHAPES[w], "dram_bytes": rd + wr, "dram_read": rd,
                      "dram_write": wr, "us": us}
        out.append("| %s | %s | %.1f | %.1f | %.1f | %.1f | %.1f | %.1f | %.1f | %.1f | %d |" % (
            d["kernel"], SHAPES[w], us, rd / 1e6, wr / 1e6, g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
            g("sm__throughput.avg.pct_of_peak_sustained_elapsed"), g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            g("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            g("smsp__issue_active.avg.pct_of_peak_sustained_active"), int(g("launch__registers_per_thread"))))
    open(os.path.join(PROF, "%s_ncu_full.md" % R), "w").write("\n".join(out) + "\n")
    json.dump({"round": R, "kernels": traffic}, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
    print("\n".join(out))
    if agg:
        print(open(os.path.join(PROF, "%s_ncu_launches.md" % R)).read()[:3000])


if __name__ == "__main__":
    main()
