"""Turn this round's ncu captures into the committed evidence under profiles/.

usage: python tools/ncu_to_profiles.py ROUND WORKLOAD LAUNCH_CSV [FULL_REP]

* LAUNCH_CSV: `ncu --metrics gpu__time_duration.sum --clock-control none --csv` of
  `bench.py --workload WORKLOAD` -> profiles/ROUND_launches_WORKLOAD.csv (copied) and
  a per-kernel table (launches, total, mean, share of the library's kernel time)
  in profiles/ROUND_ncu_WORKLOAD.md.  ncu serialises launches and runs them
  cold-cache, so compare SHARES with bench.py's live per-kernel table, not times.
* FULL_REP: one `ncu --set full` capture -> key metrics per captured launch
  (appended to the .md) and profiles/ROUND_traffic.json[WORKLOAD][tag] =
  mean dram__bytes_read.sum + dram__bytes_write.sum per launch, which bench.py
  reports as roofline.traffic for the dominant kernel.
"""
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

# kernel symbol -> bench.py tag (the LaunchScope tags of the library)
TAGS = [
    (r"part_scatter<\w+, \w+, \w+, (true|1)>", "shuffle_scatter"),
    (r"part_scatter", "part_scatter"),
    (r"part_hist", "part_hist"),
    (r"tile_base", "tile_base"),
    (r"hj_count", "hj_count"),
    (r"hj_write_fast", "hj_write"),
    (r"hj_write_kernel", "hj_write_multi"),
    (r"cross_rect", "cross_rect"),
    (r"band_write_kernel", "band_write"),
    (r"band_count_kernel", "band_count"),
    (r"nlj_kernel<[^>]*, (true|1)>", "nlj_write"),
    (r"nlj_kernel<[^>]*, (false|0)>", "nlj_count"),
    (r"pf_count", "pf_count"),
    (r"pf_write", "pf_write"),
    (r"bloom_build", "bloom_build"),
]
KEY_METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
]


def tag_of(name):
    for pat, t in TAGS:
        if re.search(pat, name):
            return t
    return None


def launch_table(path):
    rows = []
    with open(path) as f:
        text = "".join(l for l in f if l.startswith('"'))
    for r in csv.DictReader(io.StringIO(text)):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r["Metric Unit"]
            ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
            rows.append((r["Kernel Name"], ns))
    agg = defaultdict(lambda: [0, 0.0])
    for name, ns in rows:
        short = re.sub(r"\(.*", "", name).replace("void ", "").replace("<unnamed>::", "")
        agg[short][0] += 1
        agg[short][1] += ns
    return agg, len(rows)


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m, _ in KEY_METRICS:
            if m in hdr:
                d[m] = (r[hdr.index(m)], units[hdr.index(m)])
        res.append(d)
    return res


def to_bytes(v, u):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)


def main():
    rnd, wl, lcsv = sys.argv[1], sys.argv[2], sys.argv[3]
    rep = sys.argv[4] if len(sys.argv) > 4 else None
    os.makedirs(PROF, exist_ok=True)
    shutil.copy(lcsv, os.path.join(PROF, f"{rnd}_launches_{wl}.csv"))
    agg, n = launch_table(lcsv)
    lib = {k: v for k, v in agg.items() if not k.startswith("k_") and "at::" not in k and "elementwise" not in k}
    tot = sum(v[1] for v in lib.values())
    md = [f"# {rnd} ncu evidence, workload {wl}", "",
          f"Launch list: `{rnd}_launches_{wl}.csv` ({n} launches, `ncu --metrics gpu__time_duration.sum "
          f"--clock-control none` of `bench.py --workload {wl}`).  Library kernels only (generator and torch "
          "kernels excluded); ncu serialises and cold-starts every launch, so compare shares, not times.", "",
          "| kernel | launches | total ms | mean us | share |", "|---|---|---|---|---|"]
    for k, (c, ns) in sorted(lib.items(), key=lambda kv: -kv[1][1]):
        md.append(f"| `{k}` | {c} | {ns / 1e6:.3f} | {ns / c / 1e3:.1f} | {ns / tot:.3f} |")
    if rep:
        md += ["", f"## `ncu --set full` capture (`{os.path.basename(rep)}`)", ""]
        tj = os.path.join(PROF, f"{rnd}_traffic.json")
        traffic = json.load(open(tj)) if os.path.exists(tj) else {}
        acc = defaultdict(list)
        for d in full_metrics(rep):
            md.append(f"### `{re.sub(r'[(].*', '', d['kernel'])}`")
            md.append("")
            md.append("| metric | value |")
            md.append("|---|---|")
            for m, label in KEY_METRICS:
                if m in d:
                    md.append(f"| {label} (`{m}`) | {d[m][0]} {d[m][1]} |")
            md.append("")
            t = tag_of(d["kernel"])
            rb = to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else None
            wb = to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else None
            if t and rb is not None and wb is not None:
                # per template instantiation, so e.g. the scatter's pass-1 (no rid input)
                # and pass-2 launches weigh equally whatever the capture caught
                inst = re.sub(r"[(].*", "", d["kernel"])
                acc[t].append((inst, rb + wb))
        traffic[wl] = {}
        for t, v in acc.items():
            per = defaultdict(list)
            for inst, b in v:
                per[inst].append(b)
            means = [sum(x) / len(x) for x in per.values()]
            traffic[wl][t] = {"dram_bytes_per_launch": sum(means) / len(means), "launches_captured": len(v),
                              "instantiations": {k: sum(x) / len(x) for k, x in per.items()},
                              "report": os.path.basename(rep)}
        json.dump(traffic, open(tj, "w"), indent=1, sort_keys=True)
    with open(os.path.join(PROF, f"{rnd}_ncu_{wl}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md[:40]))


if __name__ == "__main__":
    main()
