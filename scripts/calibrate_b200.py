"""Write paper_2512_23379_b200/data/paper_b200.json (latency-model spec of the B200
engine) from measured bench.py JSON lines: python scripts/calibrate_b200.py BENCH.json [more.json ...]
The 1-GPU line sets the DiT step and decode costs; lines at other GPU counts (the
scaling run) calibrate the comm constants, which otherwise stay 0 (uncalibrated)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_23379_b200 import latency as LT  # noqa: E402


def main():
    lines = []
    for p in sys.argv[1:]:
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
    out = {"source": "bench.py on B200 (%s, %s); host signal/misc stages not modelled (0); no motion re-encode "
                     "(latent motion carry); comm constants %s" % (
                         one["config"]["workload"], one["metric"],
                         "calibrated from n_gpus=%s" % gs if len(gs) > 1 else "uncalibrated (1-GPU data only)"),
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
