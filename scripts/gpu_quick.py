"""Quick end-to-end check on a GPU box: build/setup/solve tiny + small, compare with the oracle."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import CONFIGS
import paper_1411_4356_b200 as pb
from oracle import steadystate as ss, liouvillian as lv
names = sys.argv[1:] or ["tiny", "small"]
for name in names:
    p = CONFIGS[name]
    t = time.time()
    s = pb.SteadyState(p)
    print(name, "build", s.build_info, flush=True)
    s.setup()
    print(name, "setup", s.setup_info, flush=True)
    s.solve()
    print(name, "solve", s.solve_info, "wall", time.time() - t, flush=True)
    rho = s.rho().cpu().numpy()
    print(name, "expect", s.expect(), flush=True)
    Lt, rhs, w, L = lv.constrained_system(p)
    rp, ci, va = pb.ss_export_matrix(s.handle, 0)
    print(name, "structure equal", np.array_equal(rp, Lt.indptr) and np.array_equal(ci, Lt.indices),
          "max val diff", np.abs(va - Lt.data).max() if len(va) == len(Lt.data) else None, "w", w, s.build_info["w_re"])
    if p.liouvillian_dim <= 40000:
        d = ss.solve_direct(p)
        print(name, "L1 diff vs direct", np.abs(rho - d).sum(), "oracle expect", ss.expect(d, p), flush=True)
    print(name, "launches", pb.ss_kernel_launches())
