"""Warp-stall samples of one ncu-captured kernel, aggregated per CUDA source line.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_ORDINAL LIB.so [top] [instance]

`instance` selects the template instantiation in the SASS (e.g. ILi8ELi1E for
fused_bf16_kernel<8, 1>; see the report's Kernel Name).

Maps each SASS address of the `--page source` view to the source line that
`nvdisasm -g` attributes to its offset inside the fused bf16 kernel
(profiling aid; needs the same .so that was profiled).
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

KERNEL = os.environ.get("NCU_KERNEL", "fused_bf16_kernel")


def line_map(lib, instance=""):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    m, cur, inside = {}, None, False
    for f in os.listdir(d):
        out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, f)], capture_output=True, text=True).stdout
        for ln in out.splitlines():
            if ln.startswith(".text.") or ln.startswith("//---"):
                inside = KERNEL in ln and instance in ln
                continue
            if not inside:
                continue
            mm = re.search(r'//## File ".*/([^/"]+)", line (\d+)(.*)', ln)
            if mm:
                cur = f"{mm.group(1)}:{mm.group(2)}" + (" <" + mm.group(3).strip()[:40] + ">" if "inlined" in mm.group(3) else "")
                continue
            mo = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
            if mo and cur:
                m[int(mo.group(1), 16)] = cur
    return m


def main():
    rep, kid, lib = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    instance = sys.argv[5] if len(sys.argv) > 5 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-id",
                          f"::regex:{KERNEL}:{kid}"], capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(out.splitlines()[1:]) if len(r) > 10]
    h = rows[0]
    iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    seen, body = set(), []
    for r in rows[1:]:
        if r[0] in seen or not r[0].startswith("0x"):
            continue
        seen.add(r[0])
        body.append(r)
    base = int(body[0][0], 16)
    lm = line_map(lib, instance)
    agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
    total = 0
    for r in body:
        s = int(r[iS]) if r[iS].isdigit() else 0
        total += s
        a = agg[lm.get(int(r[0], 16) - base, "?")]
        a[0] += s
        a[1] += int(r[iE]) if r[iE].isdigit() else 0
        for i in stall_cols:
            if r[i].isdigit():
                a[2][h[i][6:]] += int(r[i])
    print(f"total samples {total}")
    for k, (s, e, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{s:6d} {100.0 * s / max(total, 1):5.1f}% {e:10d}  {k:50s} {st.most_common(3)}")


if __name__ == "__main__":
    main()
