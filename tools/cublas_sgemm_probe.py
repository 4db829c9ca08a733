"""Launch configuration of the library's fp32 SGEMM at 4096^3 (context for the K1 family):
run under `ncu --metrics launch__grid_size,launch__block_size,launch__registers_per_thread,
launch__shared_mem_per_block_dynamic,gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active`."""
import torch

torch.backends.cuda.matmul.allow_tf32 = False
for n in (2048, 4096):
    A = torch.rand(n, n, device="cuda") * 2 - 1
    B = torch.rand(n, n, device="cuda") * 2 - 1
    C = torch.empty(n, n, device="cuda")
    for _ in range(3):
        torch.mm(A, B, out=C)
    torch.cuda.synchronize()
