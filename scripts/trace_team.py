"""Sub-step cycle profile of the chain team (trsv.cu built with -DSSB_TEAM_PROF).

usage (GPU box): cp paper_1411_4356_b200/libss_b200_teamprof.so paper_1411_4356_b200/libss_b200.so
                 python scripts/trace_team.py NAME
Prints, per factor, the median clock64 cycles between consecutive TPROF points of warp 0
of the chain team of each block (trsv.cu: 0 block start, 1 off-chain work done (G1_k,
carry), 2 x_{k-1} read, 3 partial published, 4 partials and y'_k ready, 5 reduced, 6 x_k
released, 7 block end) and the step (same team: two blocks).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1411_4356_b200 as pb  # noqa: E402
from workloads import CONFIGS  # noqa: E402

NAMES = ["start", "offchain", "x_prev", "partial", "pready", "reduce", "release", "end"]
SLACK = [(0, 8, "start->spub"), (8, 9, "spub->gstage"), (9, 10, "gstage->g1"), (10, 11, "g1->g2carry"),
         (11, 12, "g2carry->x3wait"), (12, 13, "x3wait->g3carry"), (13, 1, "g3carry->offchain")]


def main():
    s = pb.SteadyState(CONFIGS[sys.argv[1]]).setup()
    x = torch.randn(s.n, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    out = {}
    for which, nm in ((0, "L"), (1, "U")):
        pb.ss_debug_trace_trsv(s.handle, which, x.data_ptr(), y.data_ptr())
        tr = pb.ss_debug_trace_trsv(s.handle, which, x.data_ptr(), y.data_ptr()).astype(np.int64)[8:-8]
        d = {f"{NAMES[i - 1]}->{NAMES[i]}": float(np.median(tr[:, i] - tr[:, i - 1])) for i in range(1, 8)}
        for a_, b_, nm_ in SLACK:
            d[nm_] = float(np.median(tr[:, b_] - tr[:, a_]))
        d["end->next start (same team)"] = float(np.median(tr[3:, 0] - tr[:-3, 7]))
        d["three steps (same team)"] = float(np.median(tr[3:, 0] - tr[:-3, 0]))
        out[nm] = d
    print(json.dumps(out, indent=1))
    s.close()


if __name__ == "__main__":
    main()
