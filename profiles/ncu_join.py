"""Join an ncu launch list of one tree (scripts/ncu_call.sh) with the tree's per-family work
(scripts/ncu_tree.py) -> per kernel family: ncu time (cold-cache, serialised), DRAM bytes
(dram__bytes_read + write) vs algorithmic bytes, FP64 thread instructions (DFMA + DADD +
DMUL) per computed amplitude, fp64-pipe utilisation.

    python profiles/ncu_join.py <launches.csv> <tree.json> <out.json>

bench.py reads out.json (profiles/ncu_<workload>.json) for roofline.traffic and for the
measured FP64 work of the dominant kernel."""
import collections
import json
import re
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from launch_summary import load  # noqa: E402

FP64 = ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dmul_pred_on.sum")


def main():
    csv_path, tree_path, out_path = sys.argv[1:4]
    ks = load(csv_path)
    tree = json.load(open(tree_path))
    n = tree["n_qubits"]
    fam = {(f["level"], f["pass"]): f for f in tree["families"] if f["kind"] == 0}
    leaf = max(f["level"] for f in tree["families"])
    agg = collections.defaultdict(lambda: collections.Counter())
    names = {}
    total_ns = 0.0
    for d in ks:
        t = d.get("gpu__time_duration.sum", 0.0)
        total_ns += t
        m = re.match(r"tq_pass_l(\d+)_p(\d+)(_v(\d))?c?$", d["name"])
        key = ("pass", int(m.group(1)), int(m.group(2))) if m and m.group(4) != "2" else \
              ("recompute", int(m.group(1)), int(m.group(2))) if m else ("other", d["name"], 0)
        # conditional leaf sampling: pass A = (leaf, 0), the projection = (leaf, 100),
        # stage-2 pass p = (leaf, 101 + p) -- the families tqsim_profile_tree reports
        mt = re.match(r"tq_trail_(a|b(\d+))_v(\d)c?$", d["name"])
        if mt:
            v = int(mt.group(3))
            if mt.group(1) == "a":
                key = ("pass", leaf, 0 if v == 1 else 100)
            else:
                key = ("pass", leaf, 101 + int(mt.group(2))) if v != 2 else ("recompute", leaf, 101 + int(mt.group(2)))
        elif "trail_project" in d["name"]:
            key = ("pass", leaf, 100)
        a = agg[key]
        names.setdefault(key, set()).add(d["name"])
        a["kernels_per_batch"] = len(names[key])
        a["launches"] += 1
        a["ns"] += t
        a["dram"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a["fp64"] += sum(d.get(x, 0.0) for x in FP64)
        a["dfma"] += d.get(FP64[0], 0.0)
        a["pipe_pct_x_ns"] += d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0) * t
    out = {"config": tree["config"], "source": csv_path.rsplit("/", 1)[-1], "launches": len(ks),
           "total_ncu_ms": total_ns / 1e6, "families": []}
    for key, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        r = {"kernel": ("tq_pass_l%d_p%d" % key[1:]) if key[0] == "pass" else
             ("tq_pass_l%d_p%d_v2 (leaf recompute)" % key[1:]) if key[0] == "recompute" else key[1],
             "launches": a["launches"], "ncu_ms": a["ns"] / 1e6, "ncu_share": a["ns"] / total_ns,
             "dram_bytes": a["dram"], "dram_gbs": a["dram"] / a["ns"] if a["ns"] else None,
             "fp64_thread_inst": a["fp64"], "dfma_thread_inst": a["dfma"],
             "fp64_pipe_pct": a["pipe_pct_x_ns"] / a["ns"] if a["ns"] else None}
        f = fam.get(key[1:]) if key[0] == "pass" else None
        if f:
            # the launch list may cover only part of the tree: compare per-launch averages
            # launches per family (the projection family is two kernels per batch)
            nk = a["launches"] / max(1, a["kernels_per_batch"]) if a.get("kernels_per_batch") else a["launches"]
            cover = nk / f["launches"]
            alg_cov = f["alg_bytes"] * cover
            comp_cov = f["computed_states"] * cover
            r.update({"tree_launches": f["launches"], "coverage": cover,
                      "alg_bytes_per_launch": f["alg_bytes"] / f["launches"],
                      "dram_over_alg": a["dram"] / alg_cov if alg_cov else None,
                      "fp64_inst_per_computed_amp": a["fp64"] / (comp_cov * 2 ** n) if comp_cov else None,
                      "fp64_model_per_amp": f["fp64_per_amp_model"],
                      "dram_bytes_per_launch": a["dram"] / a["launches"]})
        out["families"].append(r)
    json.dump(out, open(out_path, "w"), indent=1)
    for r in out["families"][:15]:
        print("%-34s n=%5d %9.2f ms %5.3f  DRAM %6.0f GB/s  fp64 %5.1f%%  d/alg %s  fp64/amp %s" % (
            r["kernel"][:34], r["launches"], r["ncu_ms"], r["ncu_share"], r["dram_gbs"] or 0,
            r["fp64_pipe_pct"] or 0, "%.3f" % r["dram_over_alg"] if r.get("dram_over_alg") else "-",
            "%.2f" % r["fp64_inst_per_computed_amp"] if r.get("fp64_inst_per_computed_amp") else "-"))


if __name__ == "__main__":
    main()
