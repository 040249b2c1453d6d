"""Summarise a profile_round.sh capture into profiles/ (tracked).

    python tools/summarize_ncu.py TAG CONFIG [--bench gpurun_out/TAG_bench_CONFIG.json]

Writes
  profiles/TAG_launches_CONFIG.json  per-kernel launch counts / total time from
                                     the serialised launch list, and the step's
                                     kernel shares (one apply = the 6 stages);
  profiles/TAG_ncu_trisolve_CONFIG.json  key --set full metrics of one
                                     interior-block trisolve launch;
  profiles/trisolve_traffic.json     {"config", "dram_bytes_per_launch"} read by
                                     bench.py for roofline.traffic.
"""
import csv
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def short(name):
    m = re.search(r"::(\w+?)(<[^(]*>)?\(", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ix = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(lambda: [0, 0.0])
    seq = []
    for r in rows:
        k = short(r[ix["Kernel Name"]])
        ns = float(r[ix["Metric Value"]])
        per[k][0] += 1
        per[k][1] += ns
        seq.append((k, ns))
    return per, seq


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units, vals = r[0], r[1], r[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            d[k] = {"value": vals[i], "unit": units[i]}
    return d


def main():
    tag, cfg = sys.argv[1], sys.argv[2]
    go = os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    per, seq = launches(os.path.join(go, f"{tag}_launches_{cfg}.csv"))
    # one apply step = 6 launches (d, f, s, e, d_sub, c spmv), or 5 with the
    # explicit correction (d, f, s, correct, c spmv): the last device-buffer
    # step (the e2e host-buffer calls that follow run in chunks and do not
    # match the pattern).
    names = [k for k, _ in seq]
    pat5 = ["trisolve", "sell_spmv", "trisolve", "correct_kernel", "sell_spmv"]
    pat6 = ["trisolve", "sell_spmv"] * 3
    step = []
    for i in range(len(seq) - 5, -1, -1):
        for pat in (pat5, pat6):
            if i + len(pat) <= len(seq) and all(names[i + j].startswith(pat[j])
                                                for j in range(len(pat))):
                step = seq[i:i + len(pat)]
                break
        if step:
            break
    tot = sum(ns for _, ns in step)
    summ = {
        "source": f"ncu --metrics gpu__time_duration.sum --clock-control none (serialised, "
                  f"cold cache) over python bench.py --config {cfg} --steps 2 --warmup 3",
        "per_kernel": {k: {"launches": c, "total_ms": ns / 1e6, "avg_ms": ns / c / 1e6}
                       for k, (c, ns) in sorted(per.items(), key=lambda x: -x[1][1])},
        "last_step": [{"kernel": k, "ms": ns / 1e6, "share": ns / tot} for k, ns in step],
    }
    json.dump(summ, open(os.path.join(prof, f"{tag}_launches_{cfg}.json"), "w"), indent=1)
    rep = os.path.join(go, f"{tag}_trisolve_{cfg}.ncu-rep")
    d = full(rep)
    json.dump(d, open(os.path.join(prof, f"{tag}_ncu_trisolve_{cfg}.json"), "w"), indent=1)
    rd = float(d["dram__bytes_read.sum"]["value"]) * UNIT[d["dram__bytes_read.sum"]["unit"]]
    wr = float(d["dram__bytes_write.sum"]["value"]) * UNIT[d["dram__bytes_write.sum"]["unit"]]
    tri_bytes = rd + wr
    json.dump({"config": cfg, "dram_bytes_per_launch": rd + wr,
               "source": f"profiles/{tag}_ncu_trisolve_{cfg}.json (ncu --set full, one launch)"},
              open(os.path.join(prof, "trisolve_traffic.json"), "w"), indent=1)
    rep = os.path.join(go, f"{tag}_correct_{cfg}.ncu-rep")
    if os.path.exists(rep):
        d = full(rep)
        json.dump(d, open(os.path.join(prof, f"{tag}_ncu_correct_{cfg}.json"), "w"), indent=1)
        rd = float(d["dram__bytes_read.sum"]["value"]) * UNIT[d["dram__bytes_read.sum"]["unit"]]
        wr = float(d["dram__bytes_write.sum"]["value"]) * UNIT[d["dram__bytes_write.sum"]["unit"]]
        json.dump({"config": cfg, "dram_bytes_per_launch": rd + wr,
                   "source": f"profiles/{tag}_ncu_correct_{cfg}.json (ncu --set full, one launch)"},
                  open(os.path.join(prof, "correct_traffic.json"), "w"), indent=1)
        print("correct dram bytes/launch", rd + wr)
    print(json.dumps(summ["last_step"], indent=1))
    print("trisolve dram bytes/launch", tri_bytes)


if __name__ == "__main__":
    main()
