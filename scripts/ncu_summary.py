"""Summarise an ncu --set full report: per kernel duration, DRAM bytes,
tensor/L2/L1/DRAM utilisation, SM clock (dev tool)."""
import csv, io, subprocess, sys, json

METRICS = {
    "gpu__time_duration.sum": "dur",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clk",
    "launch__registers_per_thread": "regs",
}
SCALE = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1, "cycle/nsecond": 1e9,
         "cycle/usecond": 1e6}

def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:70]}
        for m, k in METRICS.items():
            if m in h:
                i = h.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * SCALE.get(units[i], 1.0)
        res.append(d)
    return res

if __name__ == "__main__":
    res = summarise(sys.argv[1])
    for d in res:
        print(f"{d['kernel'][:48]:48s} {d.get('dur',0)*1e6:8.1f}us rd {d.get('dram_rd',0)/1e6:8.1f}MB wr {d.get('dram_wr',0)/1e6:7.1f}MB "
              f"dram {d.get('dram_pct',0):5.1f}% tc {d.get('tensor_pct',0):5.1f}% l2 {d.get('l2_pct',0):5.1f}% l1 {d.get('l1_pct',0):5.1f}% clk {d.get('sm_clk',0)/1e9:.2f}GHz")
    if len(sys.argv) > 2:
        json.dump(res, open(sys.argv[2], "w"), indent=1)
