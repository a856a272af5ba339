"""Per-kernel SASS opcode counts of a multi-kernel `ncu --set full` report
(executed warp instructions per opcode, from the source page) plus the static
tensor-core / TMA / TMEM opcodes that prove the Blackwell path:

  python scripts/sass_opcode_summary.py gpurun_out/prof_full.ncu-rep profiles/r2/sass_opcodes.md
"""
import collections
import csv
import subprocess
import sys

KEY_OPS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "LDTM", "STTM", "FHFMA", "FFMA2", "HFMA2", "FFMA", "DFMA",
           "MUFU", "LDS", "STS", "LDG", "STG", "LDGSTS", "SYNCS", "ATOMS", "REDG"]


def kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", "gpu__time_duration.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    ki = rows[0].index("Kernel Name")
    names = []
    for r in rows[2:]:
        base = r[ki].split("(")[0].replace("void ", "").replace("mca_dev::", "")
        if base not in names:
            names.append(base)
    return names


def opcodes(rep, name):
    base = name.split("<")[0]
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{base}", "--launch-count", "1", "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr_i = next((i for i, r in enumerate(rows) if "Instructions Executed" in r), None)
    if hdr_i is None:
        return collections.Counter(), 0
    hdr = rows[hdr_i]
    ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
    byop, tot = collections.Counter(), 0
    for r in rows[hdr_i + 1:]:
        if r and r[0] == "Kernel Name":   # the page repeats the kernel block: count the first only
            break
        try:
            n = int(r[ie] or 0)
        except (ValueError, IndexError):
            continue
        toks = r[src].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        byop[op] += n
        tot += n
    return byop, tot


def main(rep, md):
    lines = ["# SASS opcode summary (executed warp instructions per launch, one launch per kernel)", "",
             f"Source: `{rep.split('/')[-1]}` (scripts/profile_round.sh), read with `ncu --page source --print-source sass`.",
             "", "| kernel | warp instr | " + " | ".join(KEY_OPS) + " |", "|---" * (len(KEY_OPS) + 2) + "|"]
    for k in kernels(rep):
        byop, tot = opcodes(rep, k)
        lines.append(f"| {k} | {tot} | " + " | ".join(str(byop.get(o, 0)) for o in KEY_OPS) + " |")
    with open(md, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
