import sys, time
sys.path.insert(0, '/root/repo')
from paper_1510_07230_b200 import configs, native
for n in (40, 64, 128):
    spec = configs.config3(); spec.n = (n, n, n)
    e = native.engine_for(spec)
    w = native.random_orthonormal(e, 42)
    t = time.time()
    r = e.solve(w, "opt_par_mod", True, True, max_inner=6, n_org=1, n_diag=100)
    print(n, [round(x["energy"], 10) for x in r.records], round(time.time() - t, 2), flush=True)
    e.close()
