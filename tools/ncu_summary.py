"""Summaries for profiles/ from ncu outputs brought back in gpurun_out/.

    python tools/ncu_summary.py launches LAUNCHES.csv [TITLE]
        per-kernel share of a `ncu --metrics gpu__time_duration.sum --csv
        --log-file` launch list (cold-cache, serialised: shares, not absolutes)
    python tools/ncu_summary.py full REPORT.ncu-rep LOGITS_PER_LAUNCH [TITLE]
        the key metrics of each kernel in a `--set full` capture, plus
        thread-instructions per logit and DRAM bytes vs algorithmic
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.per_cycle_active",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1}


def short(name):
    name = re.sub(r"\(.*\)$", "", name)
    return name.replace("rlo::", "").replace("(anonymous namespace)::", "")


def launches(path, title=""):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    text = open(path).read()
    text = text[text.index('"ID"'):] if '"ID"' in text else text
    for r in csv.DictReader(io.StringIO(text)):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        k = short(r["Kernel Name"])
        tot[k] += v
        cnt[k] += 1
    all_ms = sum(tot.values())
    print(f"# {title}".rstrip())
    print(f"# total kernel time {all_ms:.1f} ms over {sum(cnt.values())} launches")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{100 * v / all_ms:6.2f}%  {v:11.3f} ms  {cnt[k]:5d} launches  {k}")


def full(rep, logits, title=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, unit = rows[0], rows[1]
    print(f"# {title}".rstrip())
    for r in rows[2:]:
        print(f"  {'Kernel Name':62s} {r[h.index('Kernel Name')]}")
        vals = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:62s} {r[i]} {unit[i]}")
                try:
                    vals[k] = float(r[i].replace(",", "")) * SCALE.get(unit[i], 1)
                except ValueError:
                    pass
        if logits and "smsp__inst_executed.sum" in vals:
            print(f"  -> thread-instructions per logit: {vals['smsp__inst_executed.sum'] * 32 / logits:.2f} "
                  f"({logits:.4g} logits per launch)")
        if "dram__bytes_read.sum" in vals and "gpu__time_duration.sum" in vals:
            ms = vals["gpu__time_duration.sum"] * {"ms": 1, "us": 1e-3, "ns": 1e-6}.get(
                unit[h.index("gpu__time_duration.sum")], 1)
            print(f"  -> DRAM read {vals['dram__bytes_read.sum'] / ms / 1e6:.0f} GB/s over the launch")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
    else:
        full(sys.argv[2], float(sys.argv[3]), sys.argv[4] if len(sys.argv) > 4 else "")
