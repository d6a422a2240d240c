"""Fine-kernel throughput vs slice size at ~fixed total work (CTAs per
cluster = T/256): separates the cross-CTA exchange cost from compute."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2110_10762_b200 as pb

steps = 200
for N in (1024, 4096, 8192, 16384, 32768, 65536, 131072):
    P = max(1, (65536 * 64) // N)
    ivp = pb.heat1d_system(N, 1.0, 0.0, 0.0, 0.0, 1.0)
    F = pb.backward_euler_propagator(ivp, 1.0 / 64 * steps / 1000, steps)
    x = torch.randn(P, N, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    F.apply_batch(x, out=y); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(3): F.apply_batch(x, out=y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    info = F.info
    print(f"N={N:7d} P={P:5d} T={info.threads_per_slice:5d} CTAs/slice={info.batch_cluster:2d} "
          f"{ms:8.3f} ms  {P*N*steps/ms/1e6:8.1f} GPt/s  us/step={ms*1e3/steps:.2f}")
