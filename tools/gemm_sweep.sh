# GEMM path sweep on representative shapes (run under gpurun)
mkdir -p gpurun_out
for f in 3 4 1; do
  for s in "10240 784 256" "256 2048 1024" "256 1024 2048" "4096 4096 4096" "1024 2048 64 256" "1024 256 256" "128 256 784" "784 256 128" "8192 256 784"; do
    timeout 120 python tools/gemm_probe.py --force $f --shape $s --iters 20 2>&1 | tail -1
  done
done > gpurun_out/gemm_sweep.txt
python - >> gpurun_out/gemm_sweep.txt <<'PY'
import torch
for tf in (False, True):
    torch.backends.cuda.matmul.allow_tf32 = tf
    for m,n,k,b in [(10240,784,256,1),(256,2048,1024,1),(4096,4096,4096,1),(1024,2048,64,256)]:
        a=torch.randn(b,m,k,device='cuda'); bb=torch.randn(b,k,n,device='cuda')
        for _ in range(3): c=a@bb
        torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20): c=a@bb
        e.record(); torch.cuda.synchronize(); ms=s.elapsed_time(e)/20
        print(f"cublas tf32={tf} {m}x{n}x{k}x{b}: {ms*1e3:.1f} us {2*m*n*k*b/ms/1e9:.1f} TFLOP/s")
PY
cat gpurun_out/gemm_sweep.txt
