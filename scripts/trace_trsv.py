"""Critical-path breakdown of the block substitution (trsv.cu) from %globaltimer stamps
(per block: start, warp-0 far done, all far done, near done, x stored, flag released).

usage: python scripts/trace_trsv.py NAME [field=value ...]
For each factor prints medians (ns) of: step (flag k-1 -> flag k), frontier latency
(flag k-1 released -> CTA of block k sees it), near part, mat-vec + store, release,
and the slack of the far part (far done - flag k-1 released; negative = early).
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
        stored_prev = tr[:-1, 4]
        d = {
            "blocks": int(tr.shape[0]),
            "total_us": float(tr[:, 5].max() / 1e3),
            "step_ns": float(np.median(tr[1:, 4] - tr[:-1, 4])),
            "far_barrier_minus_prev_store_ns": float(np.median(rel[:, 2] - stored_prev)),
            "near_done_minus_prev_store_ns": float(np.median(rel[:, 3] - stored_prev)),
            "near_ns": float(np.median(rel[:, 3] - rel[:, 2])),
            "matvec_store_ns": float(np.median(rel[:, 4] - rel[:, 3])),
            "inverse_wait_ns": float(np.median(rel[:, 6] - rel[:, 3])),
            "matvec_ns": float(np.median(rel[:, 7] - rel[:, 6])),
            "store_ns": float(np.median(rel[:, 4] - rel[:, 7])),
            "release_ns": float(np.median(rel[:, 5] - rel[:, 4])),
            "x_staged_minus_prev_store_ns": float(np.median(rel[:, 1] - stored_prev)),
            "near_done_minus_x_staged_ns": float(np.median(rel[:, 3] - rel[:, 1])),
            "far_late_frac": float(np.mean(rel[:, 2] > stored_prev)),
            "first_blocks": tr[:4].tolist(),
        }
        out[nm] = d
    print(json.dumps(out), flush=True)
    s.close()


if __name__ == "__main__":
    main()
