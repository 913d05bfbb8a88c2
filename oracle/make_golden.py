"""Generates tests/golden/ from the compiled reference (oracle/_ref/mbatch_ref).

TEST INFRASTRUCTURE ONLY.  Run in the container that has /root/reference (oracle/Makefile builds
the harness from the unmodified reference sources).  Each golden file holds, for one zoo model,
the reference compiler's artefacts (signatures, lowered plans, static blocks, stage phases) and a
set of runs (schedule trace, counters, digests of params / inputs / outputs, and for small runs
the outputs and the DFG node table) produced by the reference executor.

    python oracle/make_golden.py            # writes tests/golden/*.json.gz
"""
import gzip
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref", "mbatch_ref")
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

MODELS = ["rnn", "birnn", "treelstm", "mvrnn", "nestedrnn", "drnn", "stackrnn", "fig5"]
# BASELINE.json configs (the headline is treelstm H=512 b=64).
BASELINE = [("treelstm", 256, 8, 1), ("treelstm", 512, 64, 1), ("treelstm", 512, 64, 2),
            ("mvrnn", 128, 64, 1), ("birnn", 512, 64, 1), ("nestedrnn", 512, 64, 1),
            ("treelstm", 512, 8, 1), ("mvrnn", 128, 8, 1), ("birnn", 512, 8, 1), ("nestedrnn", 512, 8, 1)]


def dump(model, hidden, batch, seed, *flags, nodes=True, outputs=True):
    cmd = [REF, "dump", "--model", model, "--hidden", str(hidden), "--batch", str(batch), "--seed", str(seed)]
    cmd += list(flags)
    if not nodes:
        cmd.append("--no-nodes")
    if not outputs:
        cmd.append("--no-outputs")
    return json.loads(subprocess.check_output(cmd))


def run_entry(j, variant):
    e = {"hidden": j["hidden"], "batch": j["batch"], "seed": j["seed"], "variant": variant, "opts": j["opts"],
         "trace": j["trace"], "digests": j["digests"], "batched_equals_unbatched": j.get("batched_equals_unbatched")}
    if "nodes" in j:
        e["nodes"] = j["nodes"]
    if "outputs" in j:
        e["outputs"] = j["outputs"]
    return e


def main():
    if not os.path.exists(REF):
        sys.exit("build the reference harness first: make -C oracle ref")
    os.makedirs(OUT, exist_ok=True)
    for model in MODELS:
        base = dump(model, 32, 4, 1)
        g = {"model": model, "params": base["params"], "instance_inputs": base["instance_inputs"],
             "signatures": base["signatures"], "plans": base["plans"], "blocks": base["blocks"],
             "ghost_sig": base["ghost_sig"], "stage_phase": base["stage_phase"], "runs": []}
        g["runs"].append(run_entry(base, "default"))
        for sched in ("depth", "agenda"):
            for gather in ("fused", "explicit"):
                for seed in (1, 2):
                    j = dump(model, 32, 8, seed, "--scheduler", sched, "--gather", gather, nodes=False)
                    g["runs"].append(run_entry(j, f"{sched}-{gather}"))
        for flag in ("--no-hoist", "--no-phases"):
            j = dump(model, 32, 4, 3, flag)
            j_plans = j["plans"]
            e = run_entry(j, flag.strip("-"))
            e["plans"] = j_plans
            e["blocks"] = j["blocks"]
            e["stage_phase"] = j["stage_phase"]
            g["runs"].append(e)
        g["runs"].append(run_entry(dump(model, 64, 64, 5, nodes=False, outputs=False), "large-b64"))
        with gzip.open(os.path.join(OUT, f"{model}.json.gz"), "wt") as f:
            json.dump(g, f, separators=(",", ":"))
        print("wrote", model)
    base = []
    for model, hidden, batch, seed in BASELINE:
        small_out = not (model == "birnn" and batch == 64)
        j = dump(model, hidden, batch, seed, nodes=False, outputs=small_out)
        base.append(run_entry(j, "baseline") | {"model": model})
        print("baseline", model, hidden, batch, seed, j["trace"]["total_nodes"], "nodes")
    with gzip.open(os.path.join(OUT, "baseline.json.gz"), "wt") as f:
        json.dump(base, f, separators=(",", ":"))


if __name__ == "__main__":
    main()
