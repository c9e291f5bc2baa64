"""SASS instruction census of librqrcp_b200.so (cuobjdump -sass): per kernel
family, the tensor (DMMA), copy (LDGSTS / UTMALDG), shared-load width and
barrier counts.  No GPU needed.
Usage: python tools/sass_census.py > profiles/r02_sass_census.md"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1509_06820_b200", "librqrcp_b200.so")
OPS = ["DMMA", "DFMA", "LDGSTS", "UTMALDG", "LDS.128", "LDS.64", "LDS", "STS", "LDG", "STG",
       "BAR.SYNC", "SHFL", "MUFU"]


def census():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True,
                         text=True, check=True).stdout
    kern = None
    counts = collections.defaultdict(collections.Counter)
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            kern = m.group(1)
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if kern and m:
            op = m.group(1)
            base = op.split(".")[0]
            counts[kern]["total"] += 1
            for key in OPS:
                if key == "LDS.128":
                    hit = base == "LDS" and ".128" in op
                elif key == "LDS.64":
                    hit = base == "LDS" and ".64" in op
                elif key == "LDS":
                    hit = base == "LDS" and ".128" not in op and ".64" not in op
                elif key == "BAR.SYNC":
                    hit = op.startswith("BAR.SYNC") or op == "BAR"
                else:
                    hit = base == key
                if hit:
                    counts[kern][key] += 1
    return counts


def family(name):
    for key in ("tc_gemm_kernel", "gemm_f64_kernel", "rank_update_big_kernel", "rank_update_k_kernel",
                "rank_update_kernel", "inner_kernel", "select_reg_kernel", "select_kernel",
                "panel_fast_kernel", "panel_kernel", "block_finish_kernel", "t_inverse_kernel",
                "swap_fused_kernel", "su_prep", "sample_update", "gemm_reduce_kernel"):
        if key in name:
            return key
    return "other"


def main():
    counts = census()
    fam = collections.defaultdict(collections.Counter)
    nk = collections.Counter()
    for k, c in counts.items():
        f = family(k)
        fam[f].update(c)
        nk[f] += 1
    print("# SASS census of librqrcp_b200.so (sm_100a)\n")
    print("`python tools/sass_census.py` (cuobjdump -sass). Counts are static instructions "
          "summed over every instantiation of a family.\n")
    print("| family | kernels | instr | " + " | ".join(OPS) + " |")
    print("|---|---|---|" + "---|" * len(OPS))
    for f in sorted(fam, key=lambda x: -fam[x]["DMMA"]):
        c = fam[f]
        print(f"| {f} | {nk[f]} | {c['total']} | " + " | ".join(str(c[o]) for o in OPS) + " |")
    tot = collections.Counter()
    for c in fam.values():
        tot.update(c)
    print(f"\nTotals: {tot['DMMA']} DMMA.8x8x4, {tot['LDGSTS']} LDGSTS, {tot['UTMALDG']} UTMALDG, "
          f"{tot['LDS.128']} LDS.128, {tot['LDS.64']} LDS.64.")


if __name__ == "__main__":
    sys.exit(main())
