"""Regenerate profiles/traffic.json (the `roofline.traffic` source of bench.py) from the raw
ncu metrics CSV of the C4 leaf-level launches (tools/r02_final.sh's traffic pass); the
previous capture is kept under "prev".

    python tools/traffic_json.py gpurun_out/r02/final2/traffic_c4.csv profiles/r02b_traffic_c4.csv
"""
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"dram__bytes_read.sum": "dram_read_bytes", "dram__bytes_write.sum": "dram_write_bytes",
        "gpu__time_duration.sum": "ms", "sm__inst_executed_pipe_fp64.sum": "fp64_warp_inst",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
        "smsp__inst_executed.sum": "warp_inst"}


def main():
    src, keep = sys.argv[1], sys.argv[2]
    shutil.copyfile(src, os.path.join(ROOT, keep))
    rows = [r for r in csv.reader(open(src)) if len(r) == 15 and r[0] != "ID"]
    launches = {}
    for r in rows:
        kname, metric, val = r[4], r[12], float(r[14].replace(",", ""))
        e = launches.setdefault(r[0], {"kernel": kname, "grid": r[8]})
        if metric in KEYS:
            e[KEYS[metric]] = val / 1e6 if metric == "gpu__time_duration.sum" else val
    out = {}  # per kernel the longest launch (the leaf level's)
    for e in launches.values():
        short = e["kernel"].split("<")[0].replace("void ", "").strip()
        if short not in out or e.get("ms", 0) > out[short].get("ms", 0):
            out[short] = e
    path = os.path.join(ROOT, "profiles", "traffic.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    new = {"source": "ncu --metrics " + ",".join(KEYS) + " --clock-control none -k regex:'hseg_loop|hseg_adj|"
           "dinit_dense|dinit_iv84' -c 3 python tools/c4_paths.py dev 1 (final round-2 build; C4 leaf-level "
           "launches; raw CSV " + keep + ")", "c4": out,
           "prev": {"source": old.get("source"), "c4": old.get("c4")}}
    for k in ("r01", "r01_source"):
        if k in old:
            new[k] = old[k]
    json.dump(new, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
