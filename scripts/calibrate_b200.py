"""Write paper_2512_23379_b200/data/paper_b200.json (latency-model spec of the B200
engine) from measured bench.py JSON lines: python scripts/calibrate_b200.py BENCH.json [more.json ...]
The 1-GPU line sets the DiT step and decode costs; lines at other GPU counts (the
scaling run) calibrate the comm constants. Without them (--estimate-comm) the comm constants
come from a byte model of the Ulysses / split-VAE exchanges at the pool's measured NVLink
peer-copy bandwidth (770 GB/s per direction, B200_PROFILING.md) plus the device-barrier
latency, at g = 8, and the spec says ESTIMATED."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_23379_b200 import latency as LT  # noqa: E402


NVLINK_GBS = 770.0        # measured peer copy per direction (B200 pool, profiling guide)
BARRIER_US = 8.0          # one stream-ordered peer barrier (flag store + acquire spin), estimate


def estimate_comm(g=8, L=10530, m=5120, heads=40, layers=40, latent_px=(416, 720), vae_halo_convs=30):
    """Per-DiT-step and per-decode comm cost at g ranks (ms): Ulysses moves q|k|v (3 m bf16 per
    token) and the attention output (m per token), each (g-1)/g of the local shard, plus the x0
    all-gather; 3 barriers per layer. The VAE pays two barriers + two edge-row copies per 3x3 conv
    and the 28-frame RGB8 gather into rank 0."""
    Ls = -(-L // g)
    per_layer = Ls * (3 * m + m) * 2 * (g - 1) / g
    step_bytes = layers * per_layer + L * 64 * 4
    dit = step_bytes / (NVLINK_GBS * 1e9) * 1e3 + layers * 3 * BARRIER_US * 1e-3
    frames = 28 * latent_px[0] * latent_px[1] * 3
    vae = frames / (NVLINK_GBS * 1e9) * 1e3 + vae_halo_convs * 2 * BARRIER_US * 1e-3
    return dit, vae


def main():
    estimate = "--estimate-comm" in sys.argv
    lines = []
    for p in [a for a in sys.argv[1:] if not a.startswith("--")]:
        for ln in open(p):
            ln = ln.strip()
            if ln.startswith("{"):
                d = json.loads(ln)
                if "components_ms" in d and d.get("impl") != "reference":
                    lines.append(d)
    base = LT.PipelineSpec(gpu_count=1, audio_ms=0.0, misc_ms=0.0)
    spec = LT.spec_from_bench(lines, base)
    one = [d for d in lines if d["n_gpus"] == 1][0]
    gs = sorted({d["n_gpus"] for d in lines})
    if len(gs) > 1:
        how = "calibrated from n_gpus=%s" % gs
    elif estimate:
        from dataclasses import replace
        dit_c, vae_c = estimate_comm()
        spec = replace(spec, dit_comm_ms=dit_c, vae_decode_comm_ms=vae_c)
        how = ("ESTIMATED, not measured: byte model of the g=8 Ulysses exchanges and split-VAE halos / frame "
               "gather at the pool's measured %.0f GB/s NVLink peer copy + %.0f us per device barrier "
               "(scripts/calibrate_b200.py estimate_comm)" % (NVLINK_GBS, BARRIER_US))
    else:
        how = "uncalibrated (1-GPU data only)"
    out = {"source": "bench.py on B200 (%s, %s); host signal/misc stages not modelled (0); no motion re-encode "
                     "(latent motion carry); comm constants %s" % (one["config"]["workload"], one["metric"], how),
           "spec": {k: getattr(spec, k) for k in LT.spec_fields()},
           "measured": {"table_component_ms": {"dit_step": {str(d["n_gpus"]): d["components_ms"]["denoise"] /
                                                            d["components_ms"].get("steps_per_chunk", 4)
                                                            for d in lines},
                                               "vae_decode": {str(d["n_gpus"]): d["components_ms"]["decode"]
                                                              for d in lines}},
                        "bench_line_1gpu": {k: one[k] for k in ("metric", "value", "unit", "ms_per_step",
                                                                "components_ms", "clocks")}}}
    path = os.path.join(os.path.dirname(LT.__file__), "data", "paper_b200.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)
    print(json.dumps(LT.predict(spec).to_dict()))


if __name__ == "__main__":
    main()
