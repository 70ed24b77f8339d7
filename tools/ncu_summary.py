"""Summarise an `ncu --set full` report (read here, no GPU) into a JSON file under profiles/.

  python tools/ncu_summary.py gpurun_out/prof_cfg2.ncu-rep profiles/ncu_r01_cfg2_summary.json \
      --batch 4096 --note "..."

Per kernel: duration, DRAM bytes read/written (per launch), DRAM throughput, fp64 pipe
and shared-memory utilisation, occupancy limits, registers.  bench.py reads
`dram_bytes_per_launch` from these files for the roofline `traffic` field.
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__occupancy_limit_registers": "occ_limit_regs",
    "launch__occupancy_limit_shared_mem": "occ_limit_smem",
    "launch__grid_size": "grid",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0}


def short(name: str) -> str:
    n = name.split("(")[0].strip()
    if n.startswith("void "):
        n = n[5:]
    return n.split("<")[0].split("::")[-1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {"source": args.rep, "note": args.note, "batch": args.batch}
    for r in rows[2:]:
        name = short(r[hdr.index("Kernel Name")])
        d = {}
        for k, lab in KEYS.items():
            if k not in hdr:
                continue
            i = hdr.index(k)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            if v != v:  # nan
                continue
            u = units[i]
            if u in SCALE:
                v *= SCALE[u]
                u = "s" if u in ("ns", "us", "usecond", "ms", "msecond", "second") else "B" if "byte" in u else u
            d[lab] = v
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes_per_launch"] = d["dram_read"] + d["dram_write"]
            if d.get("duration"):
                d["dram_gbs"] = d["dram_bytes_per_launch"] / d["duration"] / 1e9
        d["batch"] = args.batch
        out.setdefault("kernels", {})
        key = name
        n = 2
        while key in out["kernels"]:
            key = f"{name}#{n}"
            n += 1
        out["kernels"][key] = d
        if name not in out:
            out[name] = d
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps({k: {kk: v.get(kk) for kk in ("duration", "dram_bytes_per_launch", "dram_gbs", "fp64_pipe_pct")}
                      for k, v in out["kernels"].items()}, indent=1))


if __name__ == "__main__":
    main()
