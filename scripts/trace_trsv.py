"""Critical-path breakdown of the block substitution (trsv.cu) from %globaltimer stamps
(per block: chain data ready, near done, mat-vec done, x stored; helper far published;
producer saw the flag; frontier published; helper start).

usage: python scripts/trace_trsv.py NAME [field=value ...]
For each factor prints medians (ns) of the chain step and its parts, and how far the
helpers run ahead of the chain.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1411_4356_b200 as pb  # noqa: E402
from workloads import CONFIGS  # noqa: E402


def main():
    p = CONFIGS[sys.argv[1]]
    for kv in sys.argv[2:]:
        k, v = kv.split("=")
        p = p.with_(**{k: type(getattr(p, k))(float(v))})
    s = pb.SteadyState(p).setup()
    x = torch.randn(s.n, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    out = {"name": sys.argv[1], "setup": s.setup_info}
    for which, nm in ((0, "L"), (1, "U")):
        pb.ss_debug_trace_trsv(s.handle, which, x.data_ptr(), y.data_ptr())   # warm
        tr = pb.ss_debug_trace_trsv(s.handle, which, x.data_ptr(), y.data_ptr()).astype(np.int64)
        t0 = tr[:, 0].min()
        tr = tr - t0
        rel = tr[1:, :]
        prev = tr[:-1, 5]
        done_prev = tr[:-1, 3]
        med = lambda v: float(np.median(v))
        d = {
            "blocks": int(tr.shape[0]),
            "total_us": float(tr[:, 3].max() / 1e3),
            "step_ns": med(tr[1:, 3] - tr[:-1, 3]),
            "team_barrier_minus_prev_done_ns": med(rel[:, 0] - done_prev),
            "team_reduce_publish_ns": med(tr[:, 3] - tr[:, 0]),
            "y_done_minus_prev_done_ns": med(rel[:, 1] - done_prev),
            "y_late_frac": float(np.mean(rel[:, 1] > rel[:, 0])),
            "y_start_minus_prev_done_ns": med(rel[:, 2] - done_prev),
            "y_near_and_pbar_ns": med(tr[:, 6] - tr[:, 2]),
            "y_rest_ns": med(tr[:, 1] - tr[:, 6]),
            "y_start_minus_prev_y_done_ns": med(tr[1:, 2] - tr[:-1, 1]),
            "lieutenant_start_minus_prev_done_ns": med(rel[:, 7] - done_prev),
            "helper_publish_minus_prev_done_ns": med(rel[:, 4] - done_prev),
            "chain_waited_on_helpers_frac": float(np.mean(rel[:, 5] > done_prev)),
            "first_blocks": tr[:3].tolist(),
        }
        out[nm] = d
    print(json.dumps(out), flush=True)
    s.close()


if __name__ == "__main__":
    main()
