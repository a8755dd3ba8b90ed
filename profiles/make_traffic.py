"""profiles/ncu_traffic.json from ncu --set full captures: DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) and duration per launch of
each library kernel, keyed by the names bench.py reports (_lib.KERNEL_NAMES),
plus the compute-side counters bench.py quotes as the compositing kernels'
roofline: FP64-pipe and issue utilisation, active warps, threads per
instruction, shared-memory wavefronts and registers.

    python profiles/make_traffic.py OUT.json CAPTURE.ncu-rep [CAPTURE2.ncu-rep ...]
"""
import csv
import json
import subprocess
import sys

NAMES = [("k_walk<1", "k_walk<kContrib>"), ("k_replay<4", "k_replay<kGrad>"), ("k_replay<3", "k_replay<kGSum>"),
         ("k_grad_geometry", "k_grad_geometry"), ("k_project_init", None), ("k_project_planes", None), ("k_project", "k_project"), ("k_segsum", "k_segsum"),
         ("k_splat_finish", None), ("k_splat", "k_splat"), ("k_grad_image", "k_grad_image"),
         ("k_gather_prim", "k_gather_prim"), ("k_count_emit", "k_count_emit"), ("k_onesweep", "k_onesweep")]


COMPUTE = {
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefront_pct",
    "launch__registers_per_thread": "registers",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
}


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3,
            "nsecond": 1e-3, "ns": 1e-3}.get(u, 1)


def main(out, reps):
    acc = {}
    for rep in reps:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                              "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum," + ",".join(COMPUTE)],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(txt.splitlines()))
        hdr, units = rows[0], rows[1]
        ki = hdr.index("Kernel Name")
        cols = {m: hdr.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
        for r in rows[2:]:
            kname = r[ki]
            name = next((v for k, v in NAMES if k in kname), "skip")
            if not name or name == "skip":
                continue
            v = {m: float(r[c].replace(",", "")) * unit_scale(units[c]) for m, c in cols.items()}
            a = acc.setdefault(name, {"launches": 0, "dram": 0.0, "us": 0.0})
            a["launches"] += 1
            a["dram"] += v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
            a["us"] += v["gpu__time_duration.sum"]
            for m, short in COMPUTE.items():
                if m in hdr:
                    try:
                        a.setdefault("c", {}).setdefault(short, []).append(float(r[hdr.index(m)].replace(",", "")))
                    except ValueError:
                        pass
    d = {"source": "ncu --set full --clock-control none: " + ", ".join(reps),
         "kernels": {k: {"dram_bytes_per_launch": a["dram"] / a["launches"], "us_per_launch": a["us"] / a["launches"],
                         "launches": a["launches"],
                         "compute": {s: sum(v) / len(v) for s, v in a.get("c", {}).items()}} for k, a in acc.items()}}
    with open(out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
