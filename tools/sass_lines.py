"""Per-source-line totals of an ncu SASS source page: maps each sampled SASS
instruction of a kernel to its file:line through nvdisasm's line table
(-lineinfo builds) and sums instructions executed and stall samples.

    ncu -i REP --page source --csv --print-source sass > sass.csv
    cuobjdump -xelf all OBJ ; nvdisasm -g -c CUBIN > dis.sass
    python tools/sass_lines.py sass.csv dis.sass MANGLED_KERNEL [TOP]
"""
import collections
import csv
import re
import sys


def line_table(dis, fn):
    table, cur, on = {}, None, False
    for ln in open(dis):
        if ln.startswith(".text."):
            on = ln.strip().rstrip(":") == ".text." + fn
            continue
        if not on:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            table[int(m.group(1), 16)] = cur
    return table


def main():
    sass_csv, dis, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(sass_csv)))
    h = rows[1]
    ia = h.index("Warp Stall Sampling (All Samples)")
    ie = h.index("Instructions Executed")
    data = [r for r in rows[2:] if len(r) > ie and r[0].startswith("0x")]
    base = int(data[0][0], 16)
    table = line_table(dis, fn)
    agg = collections.defaultdict(lambda: [0, 0])
    for r in data:
        key = table.get(int(r[0], 16) - base, ("?", 0))
        agg[key][0] += int(r[ie] or 0)
        agg[key][1] += int(r[ia] or 0)
    ti = sum(v[0] for v in agg.values())
    ts = sum(v[1] for v in agg.values())
    print(f"instructions {ti}, stall samples {ts}, lines {len(agg)}")
    for (f, l), (ins, smp) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{f}:{l:<5} instr {100 * ins / ti:5.1f}%  samples {100 * smp / ts:5.1f}%")


if __name__ == "__main__":
    main()
