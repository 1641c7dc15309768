set -x
O=gpurun_out
T=/tmp/ncu_r02
mkdir -p $T
NCU="ncu --set full --clock-control none --import-source on -f"
cap() {
  name=$1; k=$2; s=$3; shift 3
  $NCU -k regex:$k -s $s -c 1 -o $T/$name "$@" > $O/r02_ncu_$name.log 2>&1
  ncu -i $T/$name.ncu-rep --page raw --csv > $O/r02_ncu_$name.raw.csv 2>/dev/null
  ncu -i $T/$name.ncu-rep --page details > $O/r02_ncu_$name.details.txt 2>/dev/null
  rm -f $T/$name.ncu-rep
}
cap matvec_segments k_bucket_segments 1 python tools/matvec_sweep.py --rows 100000 --bits 0
cap mulmod_resident k_mulmod 2 python bench.py --count 200000 --steps 1 --warmup 3 --no-flr --no-matvec --no-e2e --no-api
cap powvar_resident k_powvar 1 python bench.py --count 200000 --steps 1 --warmup 3 --no-flr --no-matvec --no-e2e --no-api
cap product_resident k_product_pass 1 python bench.py --count 200000 --steps 1 --warmup 3 --no-flr --no-matvec --no-e2e --no-api
