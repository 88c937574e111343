"""Hot SASS instructions of an ncu source-page CSV (ncu -i REP --page source --csv).

    python tools/ncu_hot.py gpurun_out/prof/X.source.csv [top]

Prints the sample share of each instruction with its dominant stall reasons,
and the share per opcode, so a capture can be read here without the GUI.
"""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    data = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        try:
            n = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        st = {s: int(r[idx[s]] or 0) for s in stalls}
        data.append((r[idx["Address"]], r[idx["Source"]].strip(), n, st, int(r[idx["Instructions Executed"]] or 0)))
    tot = sum(d[2] for d in data) or 1
    print(f"total samples {tot}, instructions {len(data)}")
    by_op = collections.Counter()
    by_stall = collections.Counter()
    for a, src, n, st, ex in data:
        by_op[src.split()[0] if not src.startswith("@") else src.split()[1]] += n
        by_stall.update(st)
    print("by opcode:", ", ".join(f"{k} {v / tot:.1%}" for k, v in by_op.most_common(15)))
    print("by stall:", ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in by_stall.most_common(10)))
    for a, src, n, st, ex in sorted(data, key=lambda d: -d[2])[:top]:
        s3 = ", ".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)
        print(f"{n / tot:6.2%} {a[-5:]} {src[:60]:60s} {s3}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
