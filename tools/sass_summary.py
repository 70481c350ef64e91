"""SASS instruction summary of the hot kernels of the built library
(cuobjdump -sass), for profiles/: static opcode histogram per kernel and the
mnemonics that show the sm_100a features in use (UBLKCP = cp.async.bulk /
TMA, SYNCS = mbarrier, LDGSTS = cp.async, FFMA2/FMUL2/FADD2 = packed fp32).

    python tools/sass_summary.py [lib.so] > profiles/rNN/sass_summary.md
"""
import collections
import re
import subprocess
import sys

KERNELS = ["_Z8k_streamILi5EEv11SlmTileArgs", "_Z8k_streamILi8EEv11SlmTileArgs",
           "_Z8k_rasterILb0EEv13SlmRasterArgs", "_Z8k_rasterILb1EEv13SlmRasterArgs",
           "_Z8k_pair_mILi16EEv10SlmFwdArgs", "_Z23k_gauss_backward_packedILi16ELi0EEv11SlmBackArgsPKii"]
KEY = ["UBLKCP", "SYNCS", "LDGSTS", "FFMA2", "FMUL2", "FADD2", "LDS", "STS", "LDG", "STG", "SHFL", "DFMA", "DMUL",
       "DADD", "FFMA", "BAR", "WARPSYNC"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2409_12892_b200/libsplatlm_b200.so"
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    print(f"SASS of `{lib}` (cuobjdump -sass, static instruction counts; sm_100a)\n")
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if name not in KERNELS:
            continue
        ops = collections.Counter()
        for m in re.finditer(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", f):
            ops[m.group(1)] += 1
        tot = sum(ops.values())
        print(f"### `{name}` ({tot} instructions)")
        print("- key: " + ", ".join(f"{k} {ops.get(k, 0)}" for k in KEY))
        print("- top: " + ", ".join(f"{k} {v}" for k, v in ops.most_common(12)))
        print()


if __name__ == "__main__":
    main()
