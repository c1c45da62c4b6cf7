mkdir -p gpurun_out/pair
timeout 60 python tools/gemm_probe.py --force 6 --shape 1024 2048 64 256 --iters 5 2>&1 | tail -3
for c in 2 4 8; do PFB_PAIR_CHUNK=$c timeout 60 python tools/gemm_probe.py --force 6 --shape 4096 4096 4096 --iters 10 2>&1 | tail -1; done
PFB_PAIR_BN=128 timeout 60 python tools/gemm_probe.py --force 6 --shape 4096 4096 4096 --iters 10 2>&1 | tail -1
PFB_PAIR_BN=128 timeout 60 python tools/gemm_probe.py --force 5 --shape 4096 4096 4096 --iters 10 2>&1 | tail -1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -c 1 -o gpurun_out/pair/pair6 python tools/gemm_probe.py --force 6 --shape 4096 4096 4096 --iters 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o gpurun_out/pair/cg1_3 python tools/gemm_probe.py --force 3 --shape 4096 4096 4096 --iters 1 > /dev/null 2>&1
ls gpurun_out/pair
