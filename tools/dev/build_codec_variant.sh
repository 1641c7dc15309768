#!/bin/bash
# Development helper: a library variant with a differently compiled codec unit (5 seconds), for A/B experiments:
#   tools/dev/build_codec_variant.sh <out.so> [-DHB_ENC_BLOCKS=5 -DHB_DEC_BLOCKS=4 -DHB_DEC_NJ=4 ...]
# Needs build/obj/*.o from __graft_entry__.build().  Load the result with tools/codec_rates.py --lib <out.so>.
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
out=$(realpath -m "$1"); shift
tag=$(basename "$out" .so)
cd "$ROOT/paper_2107_13797_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Wno-deprecated-gpu-targets \
     -Xptxas -v "$@" -c -o /tmp/$tag.o hb_codec.cu 2> /tmp/$tag.log
nvcc -shared -o "$out" /tmp/$tag.o "$ROOT/build/obj/hb_ops.o" "$ROOT/build/obj/hb_capi.o" "$ROOT/build/obj/hb_rng.o"
grep -A2 "f64_wideILb0" /tmp/$tag.log | grep "spill\|Used"
