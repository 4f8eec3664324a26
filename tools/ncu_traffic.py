"""Record the vocab kernel's DRAM traffic per launch from an `ncu --set full`
capture into profiles/ncu_traffic.json, keyed by bench config and stamped with
the SASS hash of the vocab-pass kernel instantiation the capture was taken from (bench.py uses the
number as roofline.traffic only while the kernels are unchanged).

    python tools/ncu_traffic.py CFG REPORT.ncu-rep [LIB.so]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    cfg, rep = sys.argv[1], sys.argv[2]
    lib = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "paper_2506_06122_b200", "lib", "librlo.so")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, unit = rows[0], rows[1]
    got = None
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if "vocab_" not in name:
            continue
        val = {}
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            i = h.index(k)
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
                     "s": 1}.get(unit[i], 1)
            val[k] = float(r[i].replace(",", "")) * scale
        got = (name, val)
        break
    if got is None:
        sys.exit("no vocab kernel in the report")
    import bench
    name, val = got
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d[f"cfg{cfg}"] = {"bytes_per_launch": val["dram__bytes_read.sum"] + val["dram__bytes_write.sum"],
                      "dram_read": val["dram__bytes_read.sum"], "dram_write": val["dram__bytes_write.sum"],
                      "launch_s_under_ncu": val["gpu__time_duration.sum"], "kernel": name,
                      "capture": os.path.basename(rep), "kernel_sig": bench.kernel_sig(name),
                      "sass_hash": bench.kernel_sass_hash(lib, bench.kernel_sig(name))}
    json.dump(d, open(p, "w"), indent=1)
    print(json.dumps(d[f"cfg{cfg}"]))


if __name__ == "__main__":
    main()
