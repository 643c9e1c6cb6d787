python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_bem.py -q -x -k "multi or far_rules or assembly_parity" > gpurun_out/pt_b15.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pt_b15.log
for o in interleave asm_first multi; do NAT_BENCH_ORDER=$o timeout 600 python -c "
import sys, json, torch; sys.path.insert(0,'.')
import bench_secondary as S
from paper_2506_06190_b200 import nat
torch.cuda.set_device(0)
def barrier(): torch.cuda.synchronize()
def ar(ms, w): return ms, w
r = S.run_c2(nat, torch, 0, 1, None, 5, barrier, ar)
print('$o', round(r['value'],1), round(r['ms_per_step'],2), r['gmres_iters'])
"; done
cat > /tmp/c2k.py <<'PY'
import sys, torch, numpy as np; sys.path.insert(0,'.')
import nat_inputs as I
from paper_2506_06190_b200 import nat
m = I.icosphere(5); mesh = nat.Mesh.from_numpy(m.v, m.t); geo = nat.nat_mesh_prepare(mesh)
near = nat.nat_bem_near_list(mesh, geo); g = torch.from_numpy(I.neumann_rigid_z(m)[None]).cuda()
As, b = nat.nat_bem_assemble_multi(mesh, geo, near, [0.5, 2.0, 8.0], g)
for _ in range(2):
    nat.nat_kernel_timer_enable(True)
    nat.nat_bem_assemble_multi(mesh, geo, near, [0.5, 2.0, 8.0], g, A=As, rhs=b)
    sec, pairs, n = nat.nat_kernel_timer_read(nat.KTIMER_FAR)
    nat.nat_kernel_timer_enable(False)
print("multi far kernel: %.3f ms, %.3e pair-evals x wavenumbers/s, frac of R(3) = %.3f" % (1e3*sec, pairs/sec, pairs/sec/(16*148*1.965e9/(2+1/3))))
nat.nat_kernel_timer_enable(True)
for k in (0.5, 2.0, 8.0): nat.nat_bem_assemble(mesh, geo, near, k, g, A=As[0], rhs=b[0])
sec, pairs, n = nat.nat_kernel_timer_read(nat.KTIMER_FAR)
nat.nat_kernel_timer_enable(False)
print("single far kernels x3: %.3f ms, frac of R(1) = %.3f" % (1e3*sec, pairs/sec/1.551e12))
PY
timeout 300 python /tmp/c2k.py
