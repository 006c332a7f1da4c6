"""Top source lines of an `ncu --page source --csv --print-source cuda,sass` export by warp-stall
samples, with the leading stall reasons and shared-memory excess wavefronts per line."""
import csv
import sys
from collections import defaultdict


def main(path, n=25):
    rows = list(csv.reader(open(path)))
    # the CUDA-source table comes first: header row starts with "Line No"
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hi]
    col = {k: i for i, k in enumerate(h)}
    stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    out = []
    tot = 0
    for r in rows[hi + 1:]:
        if not r or r[0] in ("Line No", "File Path", "Function Name") or not r[0].isdigit():
            if r and r[0] == "Address":
                break
            continue
        try:
            smp = float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        tot += smp
        st = sorted(((float(r[col[k]] or 0), k[6:]) for k in stalls), reverse=True)[:3]
        exc = r[col["L1 Wavefronts Shared Excessive"]] if "L1 Wavefronts Shared Excessive" in col else ""
        ins = r[col["Instructions Executed"]]
        out.append((smp, r[0], r[1].strip()[:90], st, exc, ins))
    out.sort(reverse=True)
    print(f"total samples {tot:.0f}")
    for smp, ln, src, st, exc, ins in out[:n]:
        print(f"{100 * smp / tot:5.1f}% L{ln:>4} inst={ins:>10} shx={exc:>8} " + ",".join(f"{k}:{v:.0f}" for v, k in st) + f" | {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
