"""Pure-write HBM bandwidth on this B200 (fill of a 2 GiB buffer) next to copy
bandwidth -- the roofline of output-bound kernels (cfg4's F2 GEMM writes
2.15 GB and reads 0.2 GB)."""
import torch
x = torch.empty(2 ** 29, device="cuda")
y = torch.empty(2 ** 29, device="cuda")
for name, fn, nbytes in (("fill (write only)", lambda: x.fill_(1.0), 4 * 2 ** 29),
                         ("zero_ (write only)", lambda: x.zero_(), 4 * 2 ** 29),
                         ("copy (read+write)", lambda: y.copy_(x), 8 * 2 ** 29)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        st.record(); fn(); en.record(); torch.cuda.synchronize()
        best = min(best, st.elapsed_time(en))
    print(f"{name}: {nbytes / best / 1e6:.0f} GB/s")
