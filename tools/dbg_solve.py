import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import port
from paper_1510_07230_b200 import configs, native
spec = configs.small_molecule(16, 4, L=8.0, max_inner=2)
spec.algorithm = "opt_par"
u0 = port.random_orthonormal(spec)
ref = port.solve(spec, u0=u0)
for pois in ["cg", "dst"]:
    e = native.engine_for(spec)
    w = e.block_from(u0)
    got = e.solve(w, algorithm="opt_par", poisson=pois, max_inner=2, n_org=1, n_diag=100)
    print(pois, got.records[0], got.energy)
    e.close()
print('ref', ref['records'][0], ref['energy'])
# manual trial evaluation on GPU via explicit block
tau = ref['records'][0]['tau']
e = native.engine_for(spec)
u = e.block_from(u0)
e.build_hamiltonian(u)
hu = e.alloc(); e.apply_hamiltonian(u, hu)
z = e.alloc(); e.diagonal_residuals(u, hu, z)
zh = e.download(z)
trial = u0 - tau * zh
bt, bo = e.block_from(trial), e.alloc()
e.orthonormalize(bt, bo, True)
e.build_hamiltonian(bo)
print('manual gpu trial energy', e.total_energy(bo))
w_ref = port.orthonormalize(spec, trial)[0]
st = port.build_hamiltonian(spec, w_ref)
print('port trial energy', port.total_energy(spec, w_ref, st)[0])
