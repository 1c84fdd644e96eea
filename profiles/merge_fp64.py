"""Merge an ncu FP64 launch list (scripts/ncu_fp64.sh: DFMA/DADD/DMUL thread instructions of
the first launches of the selected kernels, tree order) into a family file written by
ncu_join.py from the complete time + DRAM launch list of the same config:

    python profiles/merge_fp64.py <fp64.csv> <tree.json> <families.json> <tag>

Per family present in the FP64 list: fp64_inst_per_computed_amp (FP64 thread instructions /
(computed states x 2^n) of the covered launches) and the fp64-pipe utilisation replace the
family file's values; fp64_source names the list."""
import json
import subprocess
import sys
import tempfile

csv_path, tree_path, fam_path, tag = sys.argv[1:5]
with tempfile.NamedTemporaryFile(suffix=".json") as t:
    subprocess.run([sys.executable, __file__.rsplit("/", 1)[0] + "/ncu_join.py", csv_path, tree_path, t.name],
                   check=True, capture_output=True)
    fp = {r["kernel"]: r for r in json.load(open(t.name))["families"]}
fam = json.load(open(fam_path))
for r in fam["families"]:
    f = fp.get(r["kernel"])
    if not f or not f.get("fp64_inst_per_computed_amp"):
        continue
    r["fp64_inst_per_computed_amp"] = f["fp64_inst_per_computed_amp"]
    r["fp64_pipe_pct"] = f["fp64_pipe_pct"]
    r["fp64_thread_inst"] = f["fp64_thread_inst"]
    r["dfma_thread_inst"] = f["dfma_thread_inst"]
    r["fp64_source"] = "ncu FP64 thread instructions (DFMA+DADD+DMUL) over %d launches (%s)" % (f["launches"], tag)
    print("%-20s fp64/amp %.2f  pipe %.1f%%  (%d launches)" % (r["kernel"], r["fp64_inst_per_computed_amp"],
                                                             r["fp64_pipe_pct"] or 0, f["launches"]))
json.dump(fam, open(fam_path, "w"), indent=1)
