"""Round-2 profile summaries.

  python tools/make_profiles_r2.py sass      # profiles/r2_sass_summary.txt (cuobjdump of libskl.so, no GPU needed)
  python tools/make_profiles_r2.py ncu       # from gpurun_out/r2_launches.csv + gpurun_out/r2_c2_full.ncu-rep:
                                             #   profiles/r2_launches.txt, r2_ncu_c2_summary.txt, traffic.json
  python tools/make_profiles_r2.py rep IN.ncu-rep OUT.txt "what was captured"
                                             # key metrics of every launch in one capture
"""
import csv
import json
import re
import subprocess
import sys
from collections import OrderedDict

MN = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "UTCBAR", "HMMA"]


def sass():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", "paper_2601_15473_b200/libskl.so"],
                         capture_output=True, text=True).stdout
    funcs, cur = OrderedDict(), None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = {k: 0 for k in MN}
            continue
        if cur:
            for k in MN:
                if re.search(r"\b" + k + r"\b", line):
                    funcs[cur][k] += 1
    lines = ["# r2 SASS mnemonic counts per kernel (cuobjdump -sass paper_2601_15473_b200/libskl.so, sm_100a)",
             "# UTCHMMA = tcgen05.mma, UTMALDG/UTMASTG = TMA tensor load/store, UBLKCP = bulk copy,",
             "# LDTM/STTM = tcgen05.ld/st (TMEM), HMMA = legacy mma.sync (0 on every kernel)", ""]
    for f, c in funcs.items():
        if any(c[k] for k in MN if k != "HMMA") or "kernel" in f:
            lines.append(f"{f[:110]:110s} " + " ".join(f"{k}={v}" for k, v in c.items() if v or k == "HMMA"))
    open("profiles/r2_sass_summary.txt", "w").write("\n".join(lines) + "\n")
    print(len(funcs), "functions")


def ncu():
    rows = list(csv.reader(open("gpurun_out/r2_launches.csv")))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ci = {k: i for i, k in enumerate(h)}
    conv = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h) or r[ci["Metric Name"]] != "gpu__time_duration.sum":
            continue
        agg.setdefault(r[ci["Kernel Name"]], []).append(float(r[ci["Metric Value"]].replace(",", "")) *
                                                         conv[r[ci["Metric Unit"]]])
    out = ["# r2 launch list: ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised:",
           "# compare SHARES).  command: python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep",
           "# kernel, launches, mean_us, min_us, max_us"]
    step = []
    for k, v in agg.items():
        tag = ("b2b_fwd " if "b2b_kernel<2, 1" in k else "b2b_bwd " if "b2b_kernel<2, 2" in k
               else "du_fused " if "du_kernel" in k else "")
        out.append("%s%s, %d, %.1f, %.1f, %.1f" % (tag, k[:60], len(v), sum(v) / len(v), min(v), max(v)))
        if tag:
            step.append(sum(v) / len(v))
    out.append("# c2 step (b2b_fwd + b2b_bwd + du) under ncu: %.1f us; shares %s" %
               (sum(step), ", ".join("%.1f%%" % (100 * x / sum(step)) for x in step)))
    open("profiles/r2_launches.txt", "w").write("\n".join(out) + "\n")
    print("\n".join(out[-4:]))
    o = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", "gpurun_out/r2_c2_full.ncu-rep", "--page", "raw", "--csv"],
                       capture_output=True, text=True).stdout
    rows = list(csv.reader(o.splitlines()))
    h, units = rows[0], rows[1]
    ci = {k: i for i, k in enumerate(h)}
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sector_hit_rate.pct", "gpc__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic"]
    lines = ["# r2 ncu --set full --clock-control none --import-source on (one launch each of the c2 step,",
             "# tools/one_step.py 'c2 bf16'); gpc__cycles_elapsed.avg.per_second = the SM clock during the capture", ""]
    traffic = {"_source": "profiles/r2_ncu_c2_summary.txt (ncu --set full, dram__bytes_read.sum + "
                          "dram__bytes_write.sum per launch, c2 bf16)"}
    for r in rows[2:]:
        name = r[ci["Kernel Name"]]
        tag = ("b2b_fwd" if "b2b_kernel<2, 1" in name else "b2b_bwd" if "b2b_kernel<2, 2" in name
               else "du_fused" if "du_kernel" in name else name[:30])
        lines.append("[%s] %s" % (tag, name[:100]))
        for k in keys:
            if k in ci:
                lines.append("  %s = %s %s" % (k, r[ci[k]], units[ci[k]]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        val = lambda k: float(r[ci[k]].replace(",", "")) * scale.get(units[ci[k]], 1)
        traffic[tag] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        lines.append("")
    open("profiles/r2_ncu_c2_summary.txt", "w").write("\n".join(lines))
    json.dump(traffic, open("profiles/traffic.json", "w"), indent=1)
    print(traffic)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "gpc__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
        "launch__grid_size", "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic"]


def rep(path, out, what):
    o = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", path, "--page", "raw", "--csv"],
                       capture_output=True, text=True).stdout
    rows = list(csv.reader(o.splitlines()))
    h, units = rows[0], rows[1]
    ci = {k: i for i, k in enumerate(h)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    lines = ["# ncu --set full --clock-control none --import-source on: %s" % what,
             "# (%s); dram_GBps = (dram read + write bytes) / gpu__time_duration" % path, ""]
    for r in rows[2:]:
        lines.append("[%s]" % r[ci["Kernel Name"]][:110])
        for k in KEYS:
            if k in ci:
                lines.append("  %s = %s %s" % (k, r[ci[k]], units[ci[k]]))
        val = lambda k: float(r[ci[k]].replace(",", "")) * scale.get(units[ci[k]], 1)
        us = float(r[ci["gpu__time_duration.sum"]].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "ms": 1e3,
                                                                         "msecond": 1e3}[units[ci["gpu__time_duration.sum"]]]
        lines.append("  dram_GBps = %.0f" % ((val("dram__bytes_read.sum") + val("dram__bytes_write.sum")) / us / 1e3))
        lines.append("")
    open(out, "w").write("\n".join(lines))
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    {"sass": sass, "ncu": ncu, "rep": rep}[sys.argv[1]](*sys.argv[2:])
