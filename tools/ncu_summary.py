"""Summarises ncu reports into the committed profiles/ artefacts.

  python tools/ncu_summary.py gpurun_out/r01_stream.ncu-rep ... > profiles/r01_ncu_summary.md
Also refreshes profiles/ncu_traffic.json (DRAM bytes per launch per kernel,
read by bench.py's roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")]}
        for m, short in METRICS:
            if m in hdr:
                d[short] = (row[hdr.index(m)], units[hdr.index(m)])
        res.append(d)
    return res


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    traffic_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    seen = set()
    print("| report | kernel | " + " | ".join(s for _, s in METRICS) + " |")
    print("|---" * (len(METRICS) + 2) + "|")
    for path in sys.argv[1:]:
        for d in rows(path):
            cells = []
            for _, s in METRICS:
                v = d.get(s)
                cells.append("%s %s" % v if v else "")
            name = d["kernel"].replace("(anonymous namespace)::", "").replace("|", "/")
            print("| %s | `%s` | %s |" % (os.path.basename(path), name[:90], " | ".join(cells)))
            if "dram_read" in d and "dram_write" in d:
                # per kernel: the largest launch of the reports given (a tiny
                # warm-up or edge-case launch of the same template must not
                # replace the representative one)
                key = name.split("(")[0]
                b = to_bytes(*d["dram_read"]) + to_bytes(*d["dram_write"])
                if key not in seen or b > traffic[key]["dram_bytes_per_launch"]:
                    traffic[key] = {"dram_bytes_per_launch": b, "source": os.path.basename(path)}
                    if os.environ.get("MF_CAPTURE_LABEL"):  # e.g. "round-2 capture, commit abc1234"
                        traffic[key]["captured"] = os.environ["MF_CAPTURE_LABEL"]
                    seen.add(key)
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
