"""Hot SASS lines per kernel from an ncu --page source --csv --print-source sass export.

    python tools/sass_hot.py gpurun_out/<dir>/src.csv [kernel-substring] [min_exec]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    sub = sys.argv[2] if len(sys.argv) > 2 else ""
    min_exec = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1]]
            blocks.append(cur)
        elif cur is not None:
            cur.append(r)
    seen = set()
    for b in blocks:
        if sub not in b[0] or b[0] in seen:
            continue
        seen.add(b[0])
        H = b[1]
        data = [dict(zip(H, r)) for r in b[2:] if len(r) == len(H)]
        tot_s = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
        tot_i = sum(int(d["Instructions Executed"] or 0) for d in data)
        print(b[0][:90], "samples", tot_s, "inst", tot_i)
        stalls = [k for k in H if k.startswith("stall_") and "Not Issued" not in k]
        agg = {k: sum(float(d[k] or 0) for d in data) for k in stalls}
        print(" ", sorted(((k, int(v)) for k, v in agg.items()), key=lambda x: -x[1])[:8])
        if min_exec:
            for d in data:
                n = int(d["Instructions Executed"] or 0)
                if n >= min_exec:
                    print(f"  {d['Address'][-5:]} {n:9d} {d['Warp Stall Sampling (All Samples)']:>6s}  {d['Source'][:70]}")
        else:
            top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:15]
            for d in top:
                print(f"  {d['Address'][-5:]} {d['Instructions Executed']:>9s} {d['Warp Stall Sampling (All Samples)']:>6s}  {d['Source'][:70]}")


if __name__ == "__main__":
    main()
