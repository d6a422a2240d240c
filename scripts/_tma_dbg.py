import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2110_10762_b200 as pb
os.environ["PINT_FE3D_VARIANT"] = os.environ.get("V", "12")
n = 64
h = 1.0 / (n + 1)
ivp = pb.heat3d_system(n, t_final=1.0)
F = pb.forward_euler_propagator(ivp, 3 * 0.15 * h * h, 3, dtype="float32")
x = torch.rand(2, ivp.dim, device="cuda")
y = F.apply_batch(x)
torch.cuda.synchronize()
os.environ["PINT_FE3D_VARIANT"] = "8"
y2 = F.apply_batch(x)
print("equal", torch.equal(y, y2))
