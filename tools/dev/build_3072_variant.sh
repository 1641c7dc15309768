#!/bin/bash
# Development helper: a library variant whose hb_capi unit only instantiates the shapes a 3072-bit key uses
# (-DHB_DEV_ONLY_3072: 3 minutes instead of 4.5), for A/B experiments on the (48,4) / (24,4) kernels.
#   tools/dev/build_3072_variant.sh <out.so> [extra nvcc flags, e.g. -DHB_NS_SHARED_MODULUS -DHB_NS_VOLATILE]
# Needs build/obj/*.o from __graft_entry__.build().  Load the result with tools/kernel_rates.py --lib <out.so>.
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
out=$(realpath -m "$1"); shift
tag=$(basename "$out" .so)
cd "$ROOT/paper_2107_13797_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Wno-deprecated-gpu-targets \
     -Xptxas -v -DHB_DEV_ONLY_3072 "$@" -c -o /tmp/$tag.o hb_capi.cu 2> /tmp/$tag.log
nvcc -shared -o "$out" /tmp/$tag.o "$ROOT/build/obj/hb_ops.o" "$ROOT/build/obj/hb_codec.o" "$ROOT/build/obj/hb_rng.o"
grep -A2 "k_encryptILi48\|k_decryptILi24ELi4" /tmp/$tag.log | grep "spill\|Used"
