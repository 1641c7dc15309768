#!/bin/bash
# Round-2 profiling pass (run under gpurun on ONE GPU):  bash tools/profile_r02.sh
# 1. launch list of the bench command (gpu__time_duration only: shares of the step, not absolute times)
# 2. one `--set full` capture per hot kernel, small enough that ncu's ~40 replays stay short
# Reports land in gpurun_out/; tools/ncu_summary.py condenses them into profiles/ on the build machine.
set -x
O=gpurun_out
NCU="ncu --set full --clock-control none --import-source on -f"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r02_launches.csv \
    python bench.py --steps 2 --warmup 3 --flr-rows 20000 --flr-cpu-rows 0 --api-steps 1 > $O/r02_launches_bench.log 2>&1
$NCU -k regex:k_encrypt -s 1 -c 1 -o $O/r02_encrypt python tools/kernel_rates.py --key-bits 2048 --count 37888 --only encrypt --reps 1 > $O/r02_ncu_encrypt.log 2>&1
$NCU -k regex:k_decrypt -s 1 -c 1 -o $O/r02_decrypt python tools/kernel_rates.py --key-bits 2048 --count 151552 --only decrypt --reps 1 > $O/r02_ncu_decrypt.log 2>&1
$NCU -k regex:k_encrypt -s 1 -c 1 -o $O/r02_encrypt3072 python tools/kernel_rates.py --key-bits 3072 --count 37888 --only encrypt --reps 1 > $O/r02_ncu_encrypt3072.log 2>&1
$NCU -k regex:k_decrypt -s 1 -c 1 -o $O/r02_decrypt3072 python tools/kernel_rates.py --key-bits 3072 --count 113664 --only decrypt --reps 1 > $O/r02_ncu_decrypt3072.log 2>&1
$NCU -k regex:k_encode_f64_wide -s 1 -c 1 -o $O/r02_encode python tools/codec_rates.py --count 8000000 --reps 1 > $O/r02_ncu_encode.log 2>&1
$NCU -k regex:k_decode_f64_wide -s 1 -c 1 -o $O/r02_decode python tools/codec_rates.py --count 8000000 --reps 1 > $O/r02_ncu_decode.log 2>&1
$NCU -k regex:k_bucket_segments -s 1 -c 1 -o $O/r02_matvec_segments python tools/matvec_sweep.py --rows 100000 --bits 0 > $O/r02_ncu_matvec.log 2>&1
$NCU -k regex:k_fore_gradient -c 1 -o $O/r02_fore_gradient python tools/flr_scale.py --rows 37888 --iters 1 > $O/r02_ncu_fore.log 2>&1
$NCU -k regex:k_mulmod -s 2 -c 1 -o $O/r02_mulmod_resident python bench.py --count 200000 --steps 1 --warmup 3 --no-flr --no-matvec --no-e2e --no-api > $O/r02_ncu_mulmod.log 2>&1
$NCU -k regex:k_powvar -s 1 -c 1 -o $O/r02_powvar_resident python bench.py --count 200000 --steps 1 --warmup 3 --no-flr --no-matvec --no-e2e --no-api > $O/r02_ncu_powvar.log 2>&1
ls -la $O/*.ncu-rep
