"""Parse the ncu capture of tools/prof_steps.sh (one process per config, in the order 1 2 3 4 5
3-shared; each process launches the bench step, then the split build, then the split eval) into
profiles/<round>/ncu_steps.json (every kernel, §8(d)'s counters) and profiles/traffic.json (per
config: the step's, the build's and the eval's DRAM traffic -- what bench.py reports as
roofline.traffic).

    python tools/traffic_capture.py gpurun_out/<dir>/steps.csv r02

Traffic per launch = dram__bytes_read.sum + max(dram__bytes_write.sum, 32 B x
lts__t_sectors_srcunit_tex_op_write.sum): ncu runs every kernel cold and serialised, and writes
still dirty in L2 when a kernel ends reach DRAM only later, so dram__bytes_write.sum alone
undercounts what the kernel wrote."""
import csv
import json
import os
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIG_ORDER = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "cfg3_xshared"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0, "nsecond": 1e-9}
BUILD_PREFIX = ("k1_", "k_tile", "k4_top")


def short(name):
    n = name.replace("void ", "").replace("fs::", "")
    return n.split("(")[0]


def load(path):
    kernels = OrderedDict()
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: i for i, k in enumerate(hdr)}
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        kid = int(r[ix["ID"]])
        k = kernels.setdefault(kid, {"id": kid, "pid": r[ix["Process ID"]], "kernel": short(r[ix["Kernel Name"]]),
                                     "grid": r[ix["Grid Size"]], "block": r[ix["Block Size"]]})
        unit, val = r[ix["Metric Unit"]], r[ix["Metric Value"]].replace(",", "")
        try:
            v = float(val) * UNIT.get(unit, 1.0)
        except ValueError:
            continue
        k[r[ix["Metric Name"]]] = v
    return list(kernels.values())


def traffic(k):
    w = max(k.get("dram__bytes_write.sum", 0.0), 32.0 * k.get("lts__t_sectors_srcunit_tex_op_write.sum", 0.0))
    return k.get("dram__bytes_read.sum", 0.0) + w


def summarize(ks):
    return {"kernels": [k["kernel"] for k in ks], "time_s": sum(k.get("gpu__time_duration.sum", 0.0) for k in ks),
            "dram_read": sum(k.get("dram__bytes_read.sum", 0.0) for k in ks),
            "dram_write": sum(k.get("dram__bytes_write.sum", 0.0) for k in ks),
            "l2_write_from_sm": sum(32.0 * k.get("lts__t_sectors_srcunit_tex_op_write.sum", 0.0) for k in ks),
            "traffic": sum(traffic(k) for k in ks)}


def main():
    src, rnd = sys.argv[1], sys.argv[2]
    ks = load(src)
    by_pid = OrderedDict()
    for k in ks:
        by_pid.setdefault(k["pid"], []).append(k)
    out = {"_note": "per launch, from ncu (cold, serialised): traffic = dram read + max(dram write, 32 B x L2 write "
                    "sectors from the SMs); see tools/traffic_capture.py", "_source": f"profiles/{rnd}/ncu_steps.json"}
    detail = {}
    for cfg, group in zip(CONFIG_ORDER, by_pid.values()):
        names = [k["kernel"] for k in group]
        if len(group) == 3:                       # one-kernel step, then build, then eval
            step, build, ev = group[:1], group[1:2], group[2:]
        else:                                     # split step = build + eval, then build, then eval
            half = len(group) // 2
            step, rest = group[:half], group[half:]
            nb = sum(1 for k in rest if k["kernel"].startswith(BUILD_PREFIX))
            build, ev = rest[:nb], rest[nb:]
        out[cfg] = {"step": summarize(step), "build": summarize(build), "eval": summarize(ev)}
        for key in ("step", "build", "eval"):
            out[cfg][key].update(traffic=out[cfg][key]["traffic"])
        detail[cfg] = {"launch_order": names, "kernels": group}
    os.makedirs(os.path.join(ROOT, "profiles", rnd), exist_ok=True)
    json.dump(detail, open(os.path.join(ROOT, "profiles", rnd, "ncu_steps.json"), "w"), indent=1)
    json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    for cfg in CONFIG_ORDER:
        if cfg in out:
            print(cfg, {k: (round(v["traffic"] / 1e6, 1), [x for x in v["kernels"]]) for k, v in out[cfg].items()})


if __name__ == "__main__":
    main()
