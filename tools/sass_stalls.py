"""Per-kernel SASS listing with stall samples from `ncu --page source --csv
--print-source sass` output: python tools/sass_stalls.py <full_source.csv> [kernel-substr] [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
sub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 0
kern, hdr, lines = None, None, []
blocks = []
for r in rows:
    if r and r[0] == "Kernel Name":
        if kern: blocks.append((kern, lines))
        kern, lines = r[1], []
    elif r and r[0] == "Address":
        hdr = r
    elif r and hdr:
        lines.append(r)
if kern: blocks.append((kern, lines))
for kern, lines in blocks:
    if sub not in kern: continue
    tot = sum(int(l[2]) for l in lines)
    print(f"== {kern[:100]}  total samples {tot}")
    if top:
        for l in sorted(lines, key=lambda l: -int(l[2]))[:top]:
            print(f"{int(l[2]):6d} {int(l[5]):8d}  {l[1].strip()}")
    else:
        for l in lines:
            print(f"{int(l[2]):6d} {int(l[5]):8d}  {l[1].strip()}")


def blocks_summary(lines):
    """Basic blocks (runs of equal execution count): [start index, n instrs, exec count, samples]."""
    out, cur = [], None
    for i, l in enumerate(lines):
        e = int(l[5])
        if cur is None or e != cur[2]:
            cur = [i, 0, e, 0]
            out.append(cur)
        cur[1] += 1
        cur[3] += int(l[2])
    return out
