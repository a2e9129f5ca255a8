"""Per-kernel table of an `ncu --metrics ... --csv` log (one row per launch).
usage: python tools/ncu_metrics.py LOG.csv"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith("\"")) if len(r) > 10]
hdr = rows[0]
iK, iM, iV, iID = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
d = OrderedDict()
for r in rows[1:]:
    d.setdefault(r[iID], {"k": r[iK]})[r[iM]] = r[iV]
short = {"gpu__time_duration.sum": "us", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tc%",
         "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue%", "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
         "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "smem%",
         "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed": "bankrd%", "launch__grid_size": "grid"}
print("id | kernel | " + " | ".join(short.values()))
for k, v in d.items():
    name = v["k"].replace("void xlf::<unnamed>::", "").split("(")[0][:40]
    vals = []
    for m in short:
        x = v.get(m, "")
        try:
            x = f"{float(x.replace(',', '')):.1f}"
        except ValueError:
            pass
        vals.append(x)
    print(k, "|", name, "|", " | ".join(vals))
