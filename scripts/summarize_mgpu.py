"""Summarise gpurun_out/{mgpu_parity,config_runs}.jsonl and bench_n{2,4}.json."""
import json
import sys

D = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"


def lines(f):
    try:
        for ln in open(f"{D}/{f}"):
            if ln.startswith("{"):
                yield json.loads(ln)
    except FileNotFoundError:
        return


for d in lines("mgpu_parity.jsonl"):
    print(d["layout"], d["ok"], "loss", round(d["loss_rel"], 6), "grad", round(d["grad_rel"], 4),
          d["grad_rel_at"], "cos", round(d["grad_cos"], 6), "upd", round(d["upd_frac"], 4),
          "opt", round(d["opt_err"], 6))
for d in lines("config_runs.jsonl"):
    print(d["run"], round(d["tokens_per_s"]), "ms", round(d["ms_per_step"], 1), "TF/gpu",
          round(d["model_tflops_per_gpu"]), "maxmem", round(d["max_mem_gib"], 1),
          [round(x, 3) for x in d["loss_first_last"]], "offload", d["offload_acts"])
    for r in d["memory_per_rank"]:
        print("   ", r["dev"], r["share"], "alloc", round(r["max_alloc_gib"], 1), "init",
              round(r.get("init_peak_gib", 0), 1),
              "est", {k: round(v, 1) for k, v in r["estimate_gib"].items()},
              {k: (round(v, 2) if isinstance(v, float) else v) for k, v in r["executor"].items()})
for f in ("bench_n1.json", "bench_n2.json", "bench_n4.json"):
    for d in lines(f):
        c = d.get("collectives") or {}
        print(f, round(d["value"]), "e2e", round(d["e2e"]["value"]),
              "AG", c.get("allgather_v", {}).get("gbs"), "RS", c.get("reduce_scatter_v+adamw", {}).get("gbs"))
