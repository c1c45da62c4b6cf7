# ncu --set full of one kernel (regex $2, skip $3) of bench config $1 -> gpurun_out/one_<name>.ncu-rep
c=$1; k=$2; skip=${3:-0}; name=${4:-one}
export PFB_GEMM_TUNE_FILE=gpurun_out/tune_one_$c.txt
rm -f $PFB_GEMM_TUNE_FILE
timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-sweep --minimal > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k "regex:$k" -s $skip -c 1 \
  -o gpurun_out/one_$name python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --minimal --no-sweep > /dev/null 2>&1
ls -la gpurun_out/one_$name.ncu-rep
