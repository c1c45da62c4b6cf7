# compute-sanitizer memcheck over representative device paths (slow; bounded)
mkdir -p gpurun_out
export PFB_GEMM_AUTOTUNE=0
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
  python -m pytest tests/test_gpu_gemm.py -q -x -k "test_gemm_2d or feeds_batched or pair_batched or matmul_dual or small_k" \
  > gpurun_out/sanitize_gemm.log 2>&1; echo "gemm rc=$?"; tail -4 gpurun_out/sanitize_gemm.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -k "kernel_vs_reference or worked_example or concat_many or replayed" \
  > gpurun_out/sanitize_parity.log 2>&1; echo "parity rc=$?"; tail -4 gpurun_out/sanitize_parity.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
  python -m pytest tests/test_gpu_jit.py tests/test_gpu_parity.py -q -x \
  -k "hbm_scale or (specialised and (cfg2 or cfg5)) or row_strided or reduce" \
  > gpurun_out/sanitize_jit.log 2>&1; echo "jit rc=$?"; tail -4 gpurun_out/sanitize_jit.log
