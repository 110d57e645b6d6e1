"""Attribute an ncu SASS source page (instructions executed, stall samples) to kernel source lines.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
    cuobjdump -xelf all libdelimit_sm100a.so; nvdisasm -gi -fun <sym index> chain_tc.sm_100a.cubin > gi.sass
    python scripts/ncu_lines.py sass.csv gi.sass <kernel symbol> <first line> <last line> [kernel index]

Each SASS instruction's inline chain (nvdisasm -gi) is walked to the outermost frame inside the kernel body
(file chain_tc.cu, lines first..last), so inlined helpers (waits, splits, role functions) are charged to the
kernel line that calls them.  Prints the top lines by instructions executed and by stall samples, with the
opcode mix of the wait instructions.
"""
import collections
import csv
import os
import re
import sys


def parse_gi(path, sym, lo, hi):
    text = open(path).read().splitlines()
    inside, cur, out, frames, fresh = False, None, {}, [], False
    for ln in text:
        if ".text." + sym in ln and ".section" in ln:
            inside = True
            continue
        if inside and ln.strip().startswith(".section"):
            break
        if not inside:
            continue
        if "//## File" in ln:   # one inline level per line; consecutive lines form the chain of the next insn
            if not fresh:
                frames, fresh = [], True
            frames += [(f, int(l)) for f, l in re.findall(r'"([^"]+)", line (\d+)', ln)]
            # outermost frame inside [lo, hi]: the kernel-body (or chosen function) line that leads here
            inr = [l for f, l in frames if f.endswith("chain_tc.cu") and lo <= l <= hi]
            cur = inr[-1] if inr else None
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m:
            fresh = False
            out[int(m.group(1), 16)] = (cur, m.group(2))
    return out


def main():
    sass_csv, gi, sym, lo, hi = sys.argv[1:6]
    kidx = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    lo, hi = int(lo), int(hi)
    rows = list(csv.reader(open(sass_csv)))
    kernels, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"rows": []}
            kernels.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r:
            cur["rows"].append(r)
    k = kernels[kidx]
    h = k["hdr"]
    iE, iS = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    base = int(k["rows"][0][0], 16)
    lines = parse_gi(gi, sym, lo, hi)
    per_line = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
    tot_e = tot_s = 0.0
    for r in k["rows"]:
        off = int(r[0], 16) - base
        e, s = float(r[iE] or 0), float(r[iS] or 0)
        tot_e += e
        tot_s += s
        line, _ = lines.get(off, (None, ""))
        op = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip()).split()[0]
        d = per_line[line]
        d[0] += e
        d[1] += s
        d[2][op.split(".")[0]] += e
    src = open(sys.argv[7]).read().splitlines() if len(sys.argv) > 7 else None
    print(f"instructions {tot_e:.4g}, stall samples {tot_s:.0f}")
    for title, key in (("by instructions executed", 0), ("by stall samples", 1)):
        print(f"--- top lines {title}")
        for line, d in sorted(per_line.items(), key=lambda kv: -kv[1][key])[:int(os.environ.get("NCU_LINES_TOP", 28))]:
            ops = ", ".join(f"{o} {c / max(d[0], 1) * 100:.0f}%" for o, c in d[2].most_common(4))
            code = src[line - 1].strip()[:70] if (src and line) else ""
            print(f"{str(line):>6} instr {d[0] / tot_e * 100:5.1f}%  samples {d[1] / tot_s * 100:5.1f}%  [{ops}]  {code}")


if __name__ == "__main__":
    main()
