"""Per-element parity report (SURVEY §8a metric) of the tensor-core precisions against the
reference goldens, for every BASELINE run and every zoo-model golden run.  Writes JSON to argv[1].
Run on a GPU box:  python tools/parity_report.py gpurun_out/parity_report.json"""
import json
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
from conftest import MODELS, load_golden, trace_counters, trace_rows  # noqa: E402
from parity_metrics import elementwise, merge  # noqa: E402
from paper_2305_10611_b200 import mbx  # noqa: E402


def flat(j):
    if j["k"] == "t":
        return list(j["d"])
    return [x for it in j.get("items", []) for x in flat(it)]


def kw(variant):
    k = {}
    if variant.startswith("agenda"):
        k["scheduler"] = "agenda"
    if variant.endswith("explicit"):
        k["gather"] = "explicit"
    if variant == "no-hoist":
        k["hoist"] = False
    if variant == "no-phases":
        k["phases"] = False
    return k


def one(model, run, prec):
    c = mbx.Context(0, prec)
    m = mbx.Model(c, model, run["hidden"])
    m.make_params(run["seed"])
    t, d = m.make_inputs(run["seed"], run["batch"])
    r = m.evaluate_batch(t, d, run["batch"], record_nodes=True, **kw(run.get("variant", "")))
    sched = trace_rows(r.trace) == trace_rows(run["trace"]) and trace_counters(r.trace) == trace_counters(run["trace"])
    if "outputs" in run:
        want = [np.array(flat(o), np.float32) for o in run["outputs"]]
    else:
        c2 = mbx.Context(0, "fp32")
        m2 = mbx.Model(c2, model, run["hidden"])
        m2.make_params(run["seed"])
        want = [mbx.flatten_floats(o) for o in m2.evaluate_batch(t, d, run["batch"], **kw(run.get("variant", ""))).outputs]
    st = merge([elementwise(mbx.flatten_floats(r.outputs[i]), w, 1e-3) for i, w in enumerate(want)])
    st["schedule_equal"] = bool(sched)
    return st


def main():
    out = []
    for idx, run in enumerate(load_golden("baseline")):
        for prec in ("bf16x3",):
            try:
                s = one(run["model"], run, prec)
            except Exception as e:  # noqa: BLE001
                s = {"error": repr(e), "tb": traceback.format_exc()[-800:]}
            s.update(model=run["model"], hidden=run["hidden"], batch=run["batch"], seed=run["seed"], variant="baseline",
                     prec=prec)
            print(json.dumps(s), flush=True)
            out.append(s)
    for model in MODELS:
        for run in load_golden(model)["runs"]:
            try:
                s = one(model, run, "bf16x3")
            except Exception as e:  # noqa: BLE001
                s = {"error": repr(e), "tb": traceback.format_exc()[-800:]}
            s.update(model=model, hidden=run["hidden"], batch=run["batch"], seed=run["seed"], variant=run["variant"],
                     prec="bf16x3")
            print(json.dumps(s), flush=True)
            out.append(s)
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
