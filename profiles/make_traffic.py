"""Per-launch DRAM traffic of the gate-pass kernels from a committed ncu launch list.

    python profiles/make_traffic.py <launches.csv> <plain bench json> <steps covered> <out.json>

The launch list (scripts/profile_gpu.sh: gpu__time_duration + dram__bytes_read/write per
launch, every launch of `bench.py --steps 1 --warmup 3 --no-e2e --no-cpu`, i.e. 3 warm-up
+ 1 timed + 1 profiled step) gives the DRAM bytes of every tq_pass_* launch; divided by
the pass launches it is bench.py's roofline.traffic (ncu replays are cold-cache per
launch, so this is an upper bound of the in-app traffic).
"""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from launch_summary import load  # noqa: E402


def main():
    csv_path, plain_path, steps, out_path = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
    ks = [k for k in load(csv_path) if k["name"].startswith("tq_pass")]
    dram = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in ks)
    plain = json.load(open(plain_path))
    rl = plain["roofline"]
    d = {"workload": plain["config"]["workload"], "launches": len(ks), "steps_covered": steps,
         "dram_bytes_per_launch": dram / len(ks),
         "alg_bytes_per_launch": rl.get("alg_bytes_per_launch"),
         "traffic_over_alg": (dram / len(ks)) / rl["alg_bytes_per_launch"] if rl.get("alg_bytes_per_launch") else None,
         "source": "ncu launch list %s (dram__bytes_read.sum + dram__bytes_write.sum over %d tq_pass launches)"
                   % (csv_path.rsplit("/", 1)[-1], len(ks))}
    json.dump(d, open(out_path, "w"), indent=1)
    print(json.dumps(d))


if __name__ == "__main__":
    main()
