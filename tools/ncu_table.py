"""Per-kernel summary table (markdown) of an ncu --set full report of the bench forward.

    python tools/ncu_table.py REPORT.ncu-rep run_block.log

`run_block.log` (tests/probes/run_block.py output) supplies the step names in launch order.
"""
import csv
import subprocess
import sys

COLS = [("grid", ["launch__grid_size"], 1.0), ("dyn smem KB", ["launch__shared_mem_per_block_dynamic"], 1.0),
        ("time us (ncu, cold)", ["gpu__time_duration.sum"], 1.0), ("DRAM read MB", ["dram__bytes_read.sum"], 1.0),
        ("DRAM write MB", ["dram__bytes_write.sum"], 1.0), ("DRAM % of peak", ["dram__bytes_read.sum.pct_of_peak_sustained_elapsed+dram__bytes_write.sum.pct_of_peak_sustained_elapsed"], 1.0),
        ("tensor pipe %", ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"], 1.0),
        ("issue active %", ["sm__issue_active.avg.pct_of_peak_sustained_elapsed"], 1.0),
        ("warp instr (M)", ["smsp__inst_executed.sum", "sm__inst_executed.sum"], 1e-6)]


def main():
    rep, log = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, body = rows[0], rows[1], rows[2:]
    names = [ln.split()[0] for ln in open(log) if ln[:1] == "b" and len(ln.split()) > 3]

    def col(cands):
        for c in cands:
            if "+" in c:
                return [col([p]) for p in c.split("+")]
            for i, x in enumerate(h):
                if x == c or x.endswith("." + c):
                    return i
        return None

    idx = [(t, col(c), s) for t, c, s in COLS]
    print("| step | " + " | ".join(t for t, _, _ in idx) + " |")
    print("|---" * (len(idx) + 1) + "|")
    for k, r in enumerate(body):
        cells = []
        for t, i, s in idx:
            if isinstance(i, list):  # sum of several percentages
                cells.append(f"{sum(float(r[j].replace(',', '') or 0) for j in i):.1f}")
                continue
            if i is None or not r[i]:
                cells.append("-")
                continue
            v = r[i].replace(",", "")
            try:
                f = float(v)
                if units[i] == "byte":
                    f /= 1e6 if "MB" in t else 1.0
                if units[i] == "usecond" or units[i] == "us" or units[i] == "nsecond":
                    f = f / 1000 if units[i] == "nsecond" else f
                cells.append(f"{f * s:.1f}" if "grid" not in t else str(int(f)))
            except ValueError:
                cells.append(v)
        print(f"| {names[k] if k < len(names) else k} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
