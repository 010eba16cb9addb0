"""Join an ncu --set full capture's SASS page (per-instruction stall samples and executed
instructions) with the line table of the kernel's cubin, and print the hottest source lines.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep paper_2011_01112_b200/libicsched.so [kernel-substring] [N]

The cubin is extracted from the library with cuobjdump -xelf; addresses are matched with
nvdisasm --print-line-info-inline (innermost inlined location of each instruction).
"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile


def sass_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    kname = rows[0][1]
    hdr = rows[1]
    return kname, hdr, rows[2:]


def line_table(lib, kname_sub):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    table = {}
    for cub in glob.glob(os.path.join(d, "*.cubin")):
        txt = subprocess.run(["nvdisasm", "--print-line-info-inline", cub], capture_output=True, text=True).stdout
        kern, cur, prev = None, None, False
        for line in txt.splitlines():
            m = re.search(r"\.text\.(\S+):", line)
            if m:
                kern = m.group(1)
            if "//##" in line:
                if not prev:
                    m = re.search(r'File "([^"]+)", line (\d+)', line)
                    cur = (os.path.basename(m.group(1)), int(m.group(2)))
                prev = True
                continue
            prev = False
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
            if m and kern and kname_sub in kern:
                table[(kern, int(m.group(1), 16))] = cur
    return table


def main():
    rep, lib = sys.argv[1], sys.argv[2]
    sub = sys.argv[3] if len(sys.argv) > 3 else "ic_"  # substring of the mangled kernel symbol
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    kname, hdr, rows = sass_rows(rep)
    # the profiled instantiation's mangled name, e.g. "void icsched::ic_dp_kernel<(int)4, (bool)0,
    # (bool)1>(icsched::Params)" -> "ic_dp_kernelILi4ELb0ELb1EE": the line table must come from
    # that kernel's own code (another instantiation has other addresses)
    m = re.search(r"::(\w+)<([^>]*)>", kname)
    if m:
        args = "".join(f"L{'i' if t == 'int' else 'b'}{v}E"
                       for t, v in re.findall(r"\((int|bool)\)(-?\d+)", m.group(2)))
        sub = f"{m.group(1)}I{args}E"
    table = line_table(lib, sub)
    kerns = sorted({k for k, _ in table})
    ia, isamp, iexe = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    base = int(rows[0][ia], 16)  # the SASS page shows virtual addresses; the cubin starts at 0
    k = kerns[0]
    samp, exe = collections.Counter(), collections.Counter()
    why = collections.defaultdict(collections.Counter)
    total = 0.0
    for r in rows:
        loc = table.get((k, int(r[ia], 16) - base), ("?", 0))
        s = float(r[isamp] or 0)
        samp[loc] += s
        total += s
        exe[loc] += float(r[iexe] or 0)
        for i, h in stall_cols:
            why[loc][h[6:]] += float(r[i] or 0)
    print(f"# {kname}: {total:.0f} stall samples; kernel symbol {k}")
    for loc, s in samp.most_common(top):
        reasons = ", ".join(f"{n} {v / max(s, 1):.0%}" for n, v in why[loc].most_common(3) if v)
        print(f"{s / total:6.1%}  inst {exe[loc]:9.3g}  {loc[0]}:{loc[1]}  [{reasons}]")


if __name__ == "__main__":
    main()
