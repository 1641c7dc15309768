#!/bin/bash
# Round-2 profiling pass (run under gpurun on ONE GPU):  bash tools/profile_r02.sh [launches]
# 1. launch list of the bench command (gpu__time_duration only: shares of the step, not absolute times)
# 2. one `--set full` capture per hot kernel, small enough that ncu's ~40 replays stay short.  The reports (60 MB
#    each with source) stay on the GPU box in /tmp; what comes back in gpurun_out/ is the raw-metric CSV and the
#    details page of each, which tools/ncu_summary.py --csv condenses into profiles/ on the build machine.
set -x
O=gpurun_out
T=/tmp/ncu_r02
mkdir -p $T
NCU="ncu --set full --clock-control none --import-source on -f"
cap() {   # cap <name> <kernel regex> <skip> <command...>
  name=$1; k=$2; s=$3; shift 3
  $NCU -k regex:$k -s $s -c 1 -o $T/$name "$@" > $O/r02_ncu_$name.log 2>&1
  ncu -i $T/$name.ncu-rep --page raw --csv > $O/r02_ncu_$name.raw.csv 2>/dev/null
  ncu -i $T/$name.ncu-rep --page details > $O/r02_ncu_$name.details.txt 2>/dev/null
  rm -f $T/$name.ncu-rep
}
if [ "$1" = "launches" ] || [ -z "$1" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r02_launches.csv \
    python bench.py --steps 2 --warmup 3 --flr-rows 20000 --flr-cpu-rows 0 --api-steps 1 > $O/r02_launches_bench.log 2>&1
fi
cap encrypt k_encrypt 1 python tools/kernel_rates.py --key-bits 2048 --count 37888 --only encrypt --reps 1
cap decrypt k_decrypt 1 python tools/kernel_rates.py --key-bits 2048 --count 151552 --only decrypt --reps 1
cap encrypt3072 k_encrypt 1 python tools/kernel_rates.py --key-bits 3072 --count 37888 --only encrypt --reps 1
cap decrypt3072 k_decrypt 1 python tools/kernel_rates.py --key-bits 3072 --count 113664 --only decrypt --reps 1
cap encode k_encode_f64_wide 1 python tools/codec_rates.py --count 8000000 --reps 1
cap decode k_decode_f64_wide 1 python tools/codec_rates.py --count 8000000 --reps 1
cap matvec_segments k_bucket_segments 1 python tools/matvec_sweep.py --rows 100000 --bits 0
cap fore_gradient k_fore_gradient 0 python tools/flr_scale.py --rows 37888 --iters 1
cap mulmod_resident k_mulmod 2 python bench.py --count 200000 --steps 1 --warmup 3 --no-flr --no-matvec --no-e2e --no-api
cap powvar_resident k_powvar 1 python bench.py --count 200000 --steps 1 --warmup 3 --no-flr --no-matvec --no-e2e --no-api
du -sh $O
