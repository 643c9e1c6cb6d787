"""C2 far assembly: one multi-wavenumber pass (ka = 0.5, 2, 8) vs three one-wavenumber passes
(kernel timer; MUFU rooflines R(3) and R(1))."""
import sys

import torch

sys.path.insert(0, ".")
import nat_inputs as I
from paper_2506_06190_b200 import nat

m = I.icosphere(5)
mesh = nat.Mesh.from_numpy(m.v, m.t)
geo = nat.nat_mesh_prepare(mesh)
near = nat.nat_bem_near_list(mesh, geo)
g = torch.from_numpy(I.neumann_rigid_z(m)[None]).cuda()
As, b = nat.nat_bem_assemble_multi(mesh, geo, near, [0.5, 2.0, 8.0], g)
for _ in range(2):
    nat.nat_kernel_timer_enable(True)
    nat.nat_bem_assemble_multi(mesh, geo, near, [0.5, 2.0, 8.0], g, A=As, rhs=b)
    sec, pairs, n = nat.nat_kernel_timer_read(nat.KTIMER_FAR)
    nat.nat_kernel_timer_enable(False)
print("multi far kernel: %.3f ms, %.3e pair-evals x wavenumbers/s, frac of R(3) = %.3f"
      % (1e3 * sec, pairs / sec, pairs / sec / (16 * 148 * 1.965e9 / (2 + 1 / 3))))
nat.nat_kernel_timer_enable(True)
for k in (0.5, 2.0, 8.0):
    nat.nat_bem_assemble(mesh, geo, near, k, g, A=As[0], rhs=b[0])
sec, pairs, n = nat.nat_kernel_timer_read(nat.KTIMER_FAR)
nat.nat_kernel_timer_enable(False)
print("single far kernels x3: %.3f ms, frac of R(1) = %.3f" % (1e3 * sec, pairs / sec / 1.551e12))
