"""Per-instruction stall summary of an ncu source page (SASS) export:
python tools/ncu_stalls.py sass.csv [top_n]. Prints the stall reasons, the
samples by opcode and the hottest instructions."""
import collections
import csv
import sys


def main(path, top=12):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Source" in r)
    start = rows.index(hdr) + 1
    si = hdr.index("Warp Stall Sampling (All Samples)")
    src = hdr.index("Source")
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    reason, byop, data = collections.Counter(), collections.Counter(), []
    for r in rows[start:]:
        if len(r) <= si or not r[si].isdigit():
            continue
        n = int(r[si])
        ops = [o for o in r[src].strip().split() if not o.startswith("@")]
        byop[ops[0].split(".")[0] if ops else "?"] += n
        st = {c[6:]: int(r[hdr.index(c)]) for c in cols if r[hdr.index(c)].isdigit() and r[hdr.index(c)] != "0"}
        data.append((n, r[src].strip()[:64], st))
        for k, v in st.items():
            reason[k] += v
    total = sum(reason.values()) or 1
    print("reasons:", ", ".join(f"{k} {v / total:.0%}" for k, v in reason.most_common(8)))
    print("by opcode:", ", ".join(f"{k} {v}" for k, v in byop.most_common(10)))
    for n, s, st in sorted(data, key=lambda x: -x[0])[:int(top)]:
        print(f"{n:7d}  {s:64s} {st}")


if __name__ == "__main__":
    main(*sys.argv[1:])
