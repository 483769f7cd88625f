"""Summarise an ncu --set full report: key throughput metrics + top stall lines."""
import csv, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum"]

def main(rep, top=20):
    rows, units = raw(rep)
    for d in rows:
        print("==", d["Kernel Name"][:60])
        for k in KEYS:
            if k in d:
                print(f"   {k} = {d[k]} {units.get(k, '')}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data = rows[2:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src = hdr.index("Source")
    tot = sum(float(r[i_s] or 0) for r in data if len(r) > i_s)
    print("   stall samples:", tot)
    for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:top]:
        print(f"   {float(r[i_s]) / tot * 100:5.1f}%  {r[i_src][:100]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
