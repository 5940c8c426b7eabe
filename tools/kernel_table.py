"""Per-kernel table from an `ncu --metrics ... --csv` log (long format: one
row per launch and metric), and the roofline.traffic refresh.

usage: python tools/kernel_table.py <ncu.csv> [--config cN --update-traffic]

Prints, per kernel name (mean over its launches): device time, DRAM bytes
read + written, achieved DRAM GB/s, L2 RED / atomic sectors and requests,
L2 throughput %, FP64 / FMA pipe % and instructions.  With
--update-traffic, the config's hot-kernel DRAM bytes per launch go into
profiles/traffic.json together with a sha256 of the library sources that
produced them, so bench.py can say whether roofline.traffic belongs to the
build being benched.
"""
import csv
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_1808_06736_b200", "libesnufft_b200.so")

COLS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("dram__bytes_read.sum", "MB rd", 1e-6),
    ("dram__bytes_write.sum", "MB wr", 1e-6),
    ("lts__t_sectors_op_red.sum", "RED sect", 1.0),
    ("lts__t_requests_op_red.sum", "RED req", 1.0),
    ("lts__t_sectors_op_atom.sum", "ATOM sect", 1.0),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %", 1.0),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1.0),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 %", 1.0),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA %", 1.0),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wf", 1.0),
    ("smsp__inst_executed.sum", "instr", 1.0),
]


def so_sha():
    """Identity of the build: sha256 over the library's SOURCES (csrc/ and
    the Makefile; nvcc output is not byte-reproducible across rebuilds)."""
    h = hashlib.sha256()
    src = os.path.join(os.path.dirname(SO), "csrc")
    for name in sorted(os.listdir(src)):
        if name.endswith((".cu", ".cuh", ".h", ".cpp")) or name == "Makefile":
            h.update(name.encode())
            with open(os.path.join(src, name), "rb") as f:
                h.update(f.read())
    return h.hexdigest()[:16]


def to_ns(unit, v):
    return v * {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1.0)


def to_bytes(unit, v):
    return v * {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1.0)


def parse(path):
    rows = list(csv.reader(open(path, errors="replace")))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    h = rows[hdr]
    ki, ii = h.index("Kernel Name"), h.index("ID")
    mi, ui, vi = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    launches, order = {}, []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("esn::", "")
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        unit, metric = r[ui], r[mi]
        if metric == "gpu__time_duration.sum":
            v = to_ns(unit, v)
        elif metric.startswith("dram__bytes"):
            v = to_bytes(unit, v)
        key = (name, r[ii])
        if key not in launches:
            launches[key] = {}
            order.append(key)
        launches[key][metric] = v
    agg, names = {}, []
    for name, _ in order:
        if name not in agg:
            agg[name] = []
            names.append(name)
    for key in order:
        agg[key[0]].append(launches[key])
    return names, agg


def mean(ls, m):
    vals = [d[m] for d in ls if m in d]
    return sum(vals) / len(vals) if vals else None


def table(path):
    names, agg = parse(path)
    out = [f"== {os.path.basename(path)}: per kernel, mean over launches"]
    hdr = f"   {'kernel':44s} {'n':>3s} " + " ".join(f"{c[1]:>10s}" for c in COLS) + f" {'GB/s':>8s}"
    out.append(hdr)
    for n in names:
        ls = agg[n]
        cells = []
        for m, _, s in COLS:
            v = mean(ls, m)
            cells.append(f"{v * s:10.4g}" if v is not None else f"{'-':>10s}")
        t = mean(ls, "gpu__time_duration.sum")
        rd, wr = mean(ls, "dram__bytes_read.sum"), mean(ls, "dram__bytes_write.sum")
        gbs = (rd + wr) / t if (t and rd is not None and wr is not None) else None
        out.append(f"   {n[:44]:44s} {len(ls):3d} " + " ".join(cells) + (f" {gbs:8.1f}" if gbs else ""))
    return names, agg, "\n".join(out)


if __name__ == "__main__":
    path = sys.argv[1]
    names, agg, txt = table(path)
    print(txt)
    if "--update-traffic" in sys.argv:
        cfg = sys.argv[sys.argv.index("--config") + 1]
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        import bench  # noqa: E402
        import cases  # noqa: E402
        hot = bench.hot_kernel_name(cases.CONFIGS[cfg])
        ls = next((agg[n] for n in names if n.startswith(hot + "<") or n == hot), None)
        if ls is None:
            sys.exit(f"no launches of {hot} in {path}")
        traffic = mean(ls, "dram__bytes_read.sum") + mean(ls, "dram__bytes_write.sum")
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        d = json.load(open(tp)) if os.path.exists(tp) else {}
        d["_doc"] = ("DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of each config's "
                     "hot kernel from `ncu --metrics` (tools/gpu_evidence.sh -> tools/kernel_table.py); "
                     "_so holds the sha256 prefix of the library sources (csrc/) each entry was measured on")
        d[cfg] = int(traffic)
        d.setdefault("_so", {})[cfg] = so_sha()
        json.dump(d, open(tp, "w"), indent=2, sort_keys=True)
        print(f"traffic[{cfg}] = {int(traffic)} ({hot}, so {d['_so'][cfg]})")
