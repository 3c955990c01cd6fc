"""Sub-step cycle profile of lieutenant 0 (trsv.cu built with -DSSB_LT_PROF).

usage (GPU box): cp paper_1411_4356_b200/libss_b200_ltprof.so paper_1411_4356_b200/libss_b200.so
                 python scripts/trace_lt.py NAME
Prints, per factor, the median clock64 cycles between consecutive LPROF points of thread 0
of lieutenant 0's team of each block (trsv.cu: 0 block start, 1 stage ready, 2 x_{k-5}
landed, 3 early part summed, 4 x_{k-4} landed, 5 late part reduced, 6 row partials
shared, 7 q sent, 8 block end) and the cycles between blocks of the same team.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1411_4356_b200 as pb  # noqa: E402
from workloads import CONFIGS  # noqa: E402

NAMES = ["start", "stage", "x_km5", "early", "x_km4", "late", "shared", "q_sent", "end"]
TEAMS = 4


def main():
    s = pb.SteadyState(CONFIGS[sys.argv[1]]).setup()
    x = torch.randn(s.n, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    out = {}
    for which, nm in ((0, "L"), (1, "U")):
        pb.ss_debug_trace_trsv(s.handle, which, x.data_ptr(), y.data_ptr())
        tr = pb.ss_debug_trace_trsv(s.handle, which, x.data_ptr(), y.data_ptr()).astype(np.int64)[8:-8]
        d = {f"{NAMES[i - 1]}->{NAMES[i]}": float(np.median(tr[:, i] - tr[:, i - 1])) for i in range(1, 9)}
        d["block period (same team)"] = float(np.median(tr[TEAMS:, 0] - tr[:-TEAMS, 0]))
        out[nm] = d
    print(json.dumps(out, indent=1))
    s.close()


if __name__ == "__main__":
    main()
