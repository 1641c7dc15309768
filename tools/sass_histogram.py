"""SASS opcode histograms of the hot kernels in the shipped library (no GPU needed: cuobjdump reads the .so).

    python tools/sass_histogram.py profiles/r02_sass_histograms.json

For every kernel named below: instruction count, the multiplier instructions (IMAD.WIDE*), shuffles, shared / global
/ local (spill) memory instructions, WARPSYNC brackets, and the ten most frequent opcodes.
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2107_13797_b200", "_lib", "libhebatch_b200.so")
KERNELS = ["k_encryptILi32ELi4", "k_encryptILi48ELi4", "k_encryptILi16ELi4", "k_decryptILi16ELi4", "k_decryptILi24ELi4",
           "k_fore_gradientILi32ELi4", "k_mulmodILi32ELi4", "k_powvarILi32ELi4", "k_product_passILi32ELi4",
           "k_bucket_segmentsILi32ELi4", "k_encode_f64_wideILb0", "k_decode_f64_wideILb0"]


def main():
    names = subprocess.run(["cuobjdump", "-elf", LIB], capture_output=True, text=True).stdout
    syms = sorted(set(re.findall(r"\.text\.(_ZN2hb\w+)", names)))
    out = {}
    for want in KERNELS:
        match = [s for s in syms if want in s]
        if not match:
            continue
        sass = subprocess.run(["cuobjdump", "-sass", "-fun", match[0], LIB], capture_output=True, text=True).stdout
        ops = collections.Counter()
        for line in sass.splitlines():
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                ops[m.group(1)] += 1
        total = sum(ops.values())
        group = lambda pred: sum(v for k, v in ops.items() if pred(k))      # noqa: E731
        out[match[0]] = {
            "instructions": total,
            "imad_wide": group(lambda k: k.startswith("IMAD.WIDE")),
            "imad_wide_x": group(lambda k: k.startswith("IMAD.WIDE.U32.X")),
            "shfl": group(lambda k: k.startswith("SHFL")),
            "warpsync": group(lambda k: k.startswith("WARPSYNC")),
            "lds_sts": group(lambda k: k.startswith("LDS") or k.startswith("STS")),
            "ldg_stg": group(lambda k: k.startswith("LDG") or k.startswith("STG")),
            "ldl_stl_spills": group(lambda k: k.startswith("LDL") or k.startswith("STL")),
            "top": ops.most_common(10),
        }
    with open(sys.argv[1], "w") as fh:
        json.dump({"library": os.path.relpath(LIB, ROOT), "arch": "sm_100a", "kernels": out}, fh, indent=1)
    for k, v in out.items():
        print(k[:60], v["instructions"], "IMAD.WIDE", v["imad_wide"], "SHFL", v["shfl"], "spill", v["ldl_stl_spills"])


if __name__ == "__main__":
    main()
