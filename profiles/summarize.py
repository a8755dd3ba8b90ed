"""Summaries of ncu outputs: launch lists (CSV) and --set full reports."""
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((d["Kernel Name"].split("(")[0][:48], float(d["Metric Value"])))
    tot = sum(v for _, v in out)
    agg = {}
    for k, v in out:
        agg[k] = agg.get(k, 0.0) + v
    print(f"total {tot / 1e3:.1f} us over {len(out)} launches")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{v / 1e3:9.1f} us {100 * v / tot:5.1f}%  {k}")


WANT = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Compute (SM) Throughput", "DRAM Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                 "Metric Unit", "ID"))
    res = {}
    for r in rows[1:]:
        if r[mi] in WANT:
            res.setdefault((r[ii], r[ki].split("(")[0]), {})[r[mi]] = f"{r[vi]} {r[ui]}"
    for k, v in res.items():
        print(k[0], k[1])
        print("   " + "; ".join(f"{m}={v[m]}" for m in WANT if m in v))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        (launches if p.endswith(".csv") else report)(p)


def source_hot(path, kernel_regex="k_walk", skip=0, top=25):
    """Per-CUDA-line stall samples (needs -lineinfo + --import-source on)."""
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", f"regex:{kernel_regex}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    lines = {}
    fname = None
    hdr = None
    stall_cols = []
    for r in csv.reader(txt.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
            continue
        try:
            s = int(r[4] or 0)
        except ValueError:
            continue
        key = (fname, int(r[0]))
        d = lines.setdefault(key, {"src": r[1].strip()[:90], "samples": 0, "stalls": {}})
        d["samples"] += s
        for i in stall_cols:
            try:
                v = int(r[i] or 0)
            except ValueError:
                v = 0
            if v:
                d["stalls"][hdr[i][6:]] = d["stalls"].get(hdr[i][6:], 0) + v
    tot = sum(d["samples"] for d in lines.values()) or 1
    print(f"{kernel_regex} launch {skip}: {tot} samples")
    for (f, ln), d in sorted(lines.items(), key=lambda x: -x[1]["samples"])[:top]:
        st = ",".join(f"{k}:{v}" for k, v in sorted(d["stalls"].items(), key=lambda x: -x[1])[:3])
        print(f"{100 * d['samples'] / tot:5.1f}% {f}:{ln:<4} {d['src']:<90} [{st}]")


def source_inst(path, kernel_regex="k_segsum", skip=0, top=25):
    """Per-CUDA-line executed warp instructions (where the instruction count goes)."""
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", f"regex:{kernel_regex}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows, fname, hdr = {}, None, None
    for r in csv.reader(txt.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
            continue
        i = hdr.index("Instructions Executed")
        try:
            v = int(r[i] or 0)
        except ValueError:
            continue
        if v:
            rows[(fname, int(r[0]))] = (v, r[1].strip()[:90])
    tot = sum(v for v, _ in rows.values()) or 1
    print(f"{kernel_regex} launch {skip}: {tot / 1e6:.1f}M warp instructions")
    for (f, ln), (v, src) in sorted(rows.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100 * v / tot:5.1f}% {v / 1e6:7.2f}M {f}:{ln:<4} {src}")
