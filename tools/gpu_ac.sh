OUT=gpurun_out/ac; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gather_many.py tests/test_gpu_parts.py tests/test_gpu_jit.py -m gpu -q -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
bash tools/ab_compare.sh
