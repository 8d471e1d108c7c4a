"""Write profiles/<round>_launches.txt (per-kernel launch-list summary of the
`ncu --metrics gpu__time_duration.sum` pass over bench.py) and
profiles/<round>_traffic.json (dram bytes per launch from the `--set full`
captures), which bench.py reads for roofline.traffic.
Usage: python scripts/ncu_extract.py r01 gpurun_out"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}


def raw(rep, metrics):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return {h: float(r[2][i].replace(",", "")) * UNIT.get(r[1][i], 1) for i, h in enumerate(r[0]) if h in metrics}


def main(tag, d):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prof = os.path.join(root, "profiles")
    os.makedirs(prof, exist_ok=True)
    rows = list(csv.reader(open(os.path.join(d, "launches.csv"))))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            per[r[ki]].append(float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1))
    ours = {k: v for k, v in per.items() if k.startswith("nrc::") or "nrc_" in k}
    frame = sum(sum(v) for v in ours.values())
    lines = [f"# ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e`",
             f"# (--metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)",
             f"{'kernel':60s} {'launches':>8s} {'mean_us':>10s} {'share_of_nrc_time':>18s}"]
    for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:60]:60s} {len(v):8d} {sum(v) / len(v):10.2f} {sum(v) / frame:18.3f}")
    others = {k: v for k, v in per.items() if k not in ours}
    for k, v in others.items():
        lines.append(f"(not ours) {k[:49]:49s} {len(v):8d} {sum(v) / len(v):10.2f}")
    open(os.path.join(prof, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    tp = os.path.join(prof, f"{tag}_traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}  # keep kernels not re-captured this time
    traffic = {k: v for k, v in traffic.items() if k != "nrc_train_kernel"}  # (pruned in round 2)
    for name, rep in [("nrc_query_ts_kernel", "prof_query.ncu-rep"), ("nrc_train_w_kernel", "prof_train.ncu-rep"),
                      ("nrc_train_w_kernel<64>", "prof_train_w.ncu-rep"), ("nrc_adam_w_kernel<64>", "prof_adam_w.ncu-rep"),
                      ("nrc_train_ws_kernel<64>", "prof_train_ws.ncu-rep")]:
        p = os.path.join(d, rep)
        if os.path.exists(p):
            m = raw(p, ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"])
            traffic[name] = {"dram_bytes_read": m["dram__bytes_read.sum"], "dram_bytes_write": m["dram__bytes_write.sum"],
                             "traffic_bytes": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
                             "duration_us": m["gpu__time_duration.sum"],
                             "source": f"ncu --set full --clock-control none, one launch ({rep})"}
    json.dump(traffic, open(os.path.join(prof, f"{tag}_traffic.json"), "w"), indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
