"""Per-kernel DRAM traffic / duration / pipe utilisation of one captured step.

usage: python tools/ncu_traffic.py REPORT.ncu-rep OUT.json [SUMMARY.txt]

REPORT is an `ncu --set full` capture of the library's kernels over one bench
step (filter `-k regex:spt::`).  Kernels are named as bench.py's per-kernel
profile names (the `prof_begin` labels in csrc/), so bench.py can attach the
measured per-launch traffic of its dominant kernel to the roofline object.
"""
import csv
import json
import re
import subprocess
import sys

# tc kinds (csrc/tc_ffn.cu: K_ROUTER .. K_DAT) -> profile names
TC_NAMES = ["tc_router", "tc_fwd1_gate_up", "tc_fwd2_down", "tc_bwd_dA", "tc_bwd_dX",
            "tc_bwd_dW1", "tc_bwd_dW2", "tc_bwd_dWR", "tc_bwd_dAT"]

METRICS = {
    "ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_ghz": "sm__cycles_elapsed.avg.per_second",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-3, "msecond": 1,
         "nsecond": 1e-6, "Ghz": 1, "GHz": 1, "Mhz": 1e-3, "MHz": 1e-3, "hz": 1e-9, "%": 1}


def profile_name(kernel):
    m = re.search(r"tc_(?:gemm|pair_gather|pair)_kernel<(?:\(int\))?(\d+)(?:, *(?:\(bool\))?\w+)?>", kernel)
    if m:
        return TC_NAMES[int(m.group(1))]
    if "combine_kernel" in kernel:
        return "combine_bwd" if re.search(r"combine_kernel<[^,]+, (?:\(bool\))?(?:1|true)>", kernel) else "combine_fwd"
    for key, name in (("topk_hist", "topk_hist"), ("bucket_scan", "bucket_scan"),
                      ("bucket_scatter", "bucket_scatter"), ("tile_sched", "tile_sched"),
                      ("gather_dgate", "gather_dgate"), ("dwr_reduce", "dwr_reduce"),
                      ("da_post", "da_post"), ("router_simt", "router_simt"),
                      ("dgate_reduce", "dgate_reduce")):
        if key in kernel:
            return name
    return kernel[:40]


def main(rep, out, summary=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(METRICS.values())], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = profile_name(d["Kernel Name"])
        vals = {}
        for k, m in METRICS.items():
            if m in d and d[m] not in ("", "n/a"):
                vals[k] = float(d[m].replace(",", "")) * SCALE.get(u.get(m, ""), 1)
        e = res.setdefault(name, {"launches": 0, "kernel": d["Kernel Name"][:80]})
        e["launches"] += 1
        for k, v in vals.items():
            e[k] = e.get(k, 0.0) + v
    for e in res.values():  # per launch
        n = e["launches"]
        for k in METRICS:
            if k in e:
                e[k] /= n
        e["dram_read_bytes"] = e.pop("dram_read", 0.0)
        e["dram_write_bytes"] = e.pop("dram_write", 0.0)
        e["ncu_ms"] = e.pop("ms", 0.0)
        if e["ncu_ms"] > 0:
            e["dram_gbs"] = (e["dram_read_bytes"] + e["dram_write_bytes"]) / e["ncu_ms"] / 1e6
    doc = {"source": f"ncu --set full --clock-control none ({rep}); per launch", "kernels": res}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    if summary:
        with open(summary, "w") as f:
            f.write(f"# {doc['source']}\n")
            f.write(f"{'kernel':18s} {'ms':>7s} {'DRAM GB':>8s} {'DRAM GB/s':>9s} {'tensor%':>8s} "
                    f"{'L2%':>6s} {'L2hit%':>7s} {'SM GHz':>7s}\n")
            for name, e in sorted(res.items(), key=lambda t: -t[1]["ncu_ms"]):
                f.write(f"{name:18s} {e['ncu_ms']:7.3f} "
                        f"{(e['dram_read_bytes'] + e['dram_write_bytes']) / 1e9:8.3f} "
                        f"{e.get('dram_gbs', 0):9.0f} {e.get('tensor_pct', 0):8.1f} "
                        f"{e.get('lts_pct', 0):6.1f} {e.get('l2_hit_pct', 0):7.1f} "
                        f"{e.get('sm_ghz', 0):7.2f}\n")
    print(json.dumps({k: round(v["ncu_ms"], 3) for k, v in res.items()}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
