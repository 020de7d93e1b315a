import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import port
from paper_1510_07230_b200 import configs, native
for spec in [configs.small_molecule(16, 4, L=8.0), configs.small_molecule(14, 4, L=8.0)]:
    u0 = port.random_orthonormal(spec)
    rng = np.random.default_rng(1)
    z = rng.standard_normal(u0.shape)
    e = native.engine_for(spec)
    bw, bz = e.block_from(u0), e.block_from(z)
    wq = np.prod(spec.spacing)
    t = u0 - 0.09 * z
    g = e.gram_lincomb(bw, -0.09, bz)
    print(spec.name, 'lincomb', np.abs(g - wq * t @ t.T).max())
    for nn in [1, 2, 4]:
        sp2 = configs.ProblemSpec("x", spec.n, spec.extent, [], nn, hartree=False, xc=False)
        e2 = native.engine_for(sp2)
        b1, b2 = e2.block_from(u0[:nn].copy()), e2.block_from(z[:nn].copy())
        g2 = e2.gram_lincomb(b1, -0.09, b2)
        tt = t[:nn]
        print('   N', nn, np.abs(g2 - wq * tt @ tt.T).max(), np.abs(e2.gram(b1, b1) - wq * u0[:nn] @ u0[:nn].T).max())
        e2.close()
    e.close()
