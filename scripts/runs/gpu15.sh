python -m paper_2506_06190_b200.build > /dev/null || exit 1
python - <<'P'
import sys, torch
sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat
m = I.icosphere(5)
mesh = nat.Mesh.from_numpy(m.v, m.t); geo = nat.nat_mesh_prepare(mesh)
smp, stri = nat.nat_mc_sample(mesh, geo, 10000, 20250606)
eps, w = nat.mc_weights(geo.total_area, 10000)
for ns in (1, 2, 3):
    p = torch.ones(ns, 10000, dtype=torch.complex128, device="cuda")
    ks = [0.5, 2.0, 8.0][:ns]
    for _ in range(3): nat.nat_mc_apply(smp, ks, p, w, eps, "fp32")
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): nat.nat_mc_apply(smp, ks, p, w, eps, "fp32")
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"mc_apply nsys={ns}: {ms*1e3:.1f} us/call -> {ns*1e8/ms/1e9:.2f} Tpair/s (incl near-list build + small kernels)")
P
