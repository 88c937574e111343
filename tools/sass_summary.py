"""SASS evidence for the tensor-core kernels (run here, on the CPU box, from the built objects).

    python tools/sass_summary.py

For each kernel: the tcgen05 / TMA / tensor instruction counts (UTCHMMA = tcgen05.mma,
LDTM / STTM = tcgen05.ld / st, UTCBAR = tcgen05.commit, SYNCS = mbarrier waits), the
opcode histogram of its hottest loop (the innermost backward branch with the most
instructions) and that loop's listing, into profiles/r02_sass_<kernel>.txt.
"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2602_24066_b200", "csrc", "build", "sigb_trunc.o")
KERNELS = {
    "trunc_pq_backward_kernel": "_ZN4sigb5trunc2pq24trunc_pq_backward_kernelILi16ELi4EEEvPKflllS4_llS4_llPf",
    "trunc_pq_backward_kernel_d8_n5": "_ZN4sigb5trunc2pq24trunc_pq_backward_kernelILi8ELi5EEEvPKflllS4_llS4_llPf",
    "trunc_tc_forward_kernel": "_ZN4sigb5trunc2tc23trunc_tc_forward_kernelILi16ELi4EEEvPKfllPflli",
}
MARKERS = ("UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTCATOMSWS", "SYNCS", "UBLKCP", "LDGSTS", "SHFL", "FFMA2", "FFMA")


def main():
    for name, mangled in KERNELS.items():
        out = subprocess.run(["cuobjdump", "-sass", "-fun", mangled, OBJ], capture_output=True, text=True).stdout
        ins = []
        for line in out.splitlines():
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        op = lambda t: re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
        total = collections.Counter(op(t) for _, t in ins)
        loops = []
        for a, t in ins:
            m = re.search(r"BRA\s+(?:`\()?(?:\.L_x_\d+)?0x([0-9a-f]+)", t)
            if m and int(m.group(1), 16) < a:
                loops.append((int(m.group(1), 16), a))
        hot = None
        for lo, hi in loops:
            body = [(a, t) for a, t in ins if lo <= a <= hi]
            nested = any(lo < l2 and h2 < hi for l2, h2 in loops)
            if any("LDTM" in t or "STTM" in t for _, t in body) and not nested:
                if hot is None or len(body) > len(hot[2]):
                    hot = (lo, hi, body)
        lines = [f"# {name} ({mangled}) from {os.path.relpath(OBJ, ROOT)}, sm_100a",
                 f"# {len(ins)} instructions",
                 "# tcgen05/TMA/tensor markers: " + ", ".join(f"{k}={sum(v for o, v in total.items() if o.startswith(k))}"
                                                              for k in MARKERS)]
        if hot:
            lo, hi, body = hot
            h = collections.Counter(op(t) for _, t in body)
            lines.append(f"# hot loop 0x{lo:x}-0x{hi:x}: {len(body)} instructions: " +
                         ", ".join(f"{k} {v}" for k, v in h.most_common(24)))
            lines += [f"{a:6x}  {t}" for a, t in body]
        path = os.path.join(ROOT, "profiles", f"r02_sass_{name}.txt")
        with open(path, "w") as f:
            f.write("\n".join(lines) + "\n")
        print(lines[2])
        if hot:
            print(lines[3][:300])


if __name__ == "__main__":
    main()
