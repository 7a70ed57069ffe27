"""Golden memory accounting and CSV exports from the REFERENCE simulator.

Build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src HETPLAN_PURE_PYTHON=1 python tests/golden/make_memory_golden.py

For every plan in plans.json (reference plan bytes), runs the unmodified
``simulate_plan`` (simulate.py:590-714) and records the per-device memory peaks
(``Timeline.memory_peaks``, exact float reprs) and the SHA-256 of the files
``Timeline.write_gantt_csv`` / ``write_memory_csv`` write (simulate.py:115-137).
tests/test_plan_parity.py::test_memory_replay_bit_exact compares the product's
restatement (plan/schedule.memory_replay, write_*_csv) byte for byte.
"""

import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))

from hetplan.configure import TrainingPlan  # noqa: E402  (reference)
from hetplan.costs import CostContext  # noqa: E402
from hetplan.partition import build_cluster_graph  # noqa: E402
from hetplan.simulate import simulate_plan  # noqa: E402
from hetplan.workload import fit_runtime_model, load_cluster_profile, load_model_workload  # noqa: E402


def _sha(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def main():
    with open(os.path.join(HERE, "plans.json")) as fh:
        cases = json.load(fh)
    out = {}
    for case in cases:
        if case.get("events") is None:
            continue
        prof = load_cluster_profile(os.path.join(HERE, case["cluster"]))
        model, workload = load_model_workload(os.path.join(HERE, case["model"]))
        ctx = CostContext(graph=build_cluster_graph(prof), runtime=fit_runtime_model(prof),
                          model=model, workload=workload)
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as fh:
            fh.write(case["plan_json"])
            plan_path = fh.name
        plan = TrainingPlan.load(plan_path, prof)
        os.unlink(plan_path)
        tl = simulate_plan(ctx, plan)
        with tempfile.TemporaryDirectory() as d:
            tl.write_gantt_csv(os.path.join(d, "g.csv"))
            tl.write_memory_csv(os.path.join(d, "m.csv"))
            out[case["name"]] = {
                "peaks": {dev: {c: repr(v) for c, v in p.items()}
                          for dev, p in sorted(tl.memory_peaks.items())},
                "gantt_sha256": _sha(os.path.join(d, "g.csv")),
                "memory_sha256": _sha(os.path.join(d, "m.csv")),
            }
    with open(os.path.join(HERE, "memory.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print(f"wrote {len(out)} cases")


if __name__ == "__main__":
    sys.exit(main())
