"""Critical-path breakdown of the block substitution (trsv.cu) from the %globaltimer
stamps of ss_debug_trace_trsv (include/ss_b200.h lists them): chain team, lieutenants,
helpers and producer per block, relative to the previous block's x being stored.

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
        step = tr[1:, 3] - tr[:-1, 3]
        ex = np.maximum(0, step - med(step))
        d = {
            "blocks": int(tr.shape[0]),
            "total_us": float(tr[:, 3].max() / 1e3),
            "step_ns": med(step),
            "step_pct_ns": [float(v) for v in np.percentile(step, [10, 50, 90, 99])],
            "excess_us": float(ex.sum() / 1e3),
            "excess_helper_late_us": float(np.sum(np.where(rel[:, 5] > done_prev - 2000, ex, 0)) / 1e3),
            # chain team of block k (relative to x_{k-1} stored)
            "team_offchain_done_ns": med(rel[:, 10] - done_prev),
            "team_read_xprev_ns": med(rel[:, 13] - done_prev),
            "team_q_landed_ns": med(rel[:, 6] - done_prev),
            "team_reduced_ns": med(rel[:, 0] - done_prev),
            "team_reduce_store_ns": med(tr[:, 3] - tr[:, 0]),
            "team_push_minus_store_ns": med(tr[:, 8] - tr[:, 3]),
            # lieutenants (relative to x_{k-1} stored)
            "lt_stage_ready_ns": med(rel[:, 12] - done_prev),
            "lt_early_done_ns": med(rel[:, 11] - done_prev),
            "lt_late_landed_ns": med(rel[:, 7] - done_prev),
            "lt_q_sent_ns": med(rel[:, 9] - done_prev),
            "lt6_q_sent_ns": med(rel[:, 2] - done_prev),
            "lt_late_landed_minus_push_km3_ns": med(tr[3:, 7] - tr[:-3, 8]),
            "lt_early_done_minus_push_km4_ns": med(tr[4:, 11] - tr[:-4, 8]),
            # helpers / producer
            "helper_publish_ns": med(rel[:, 4] - done_prev),
            "producer_flag_pct_ns": [float(v) for v in np.percentile(rel[:, 5] - done_prev, [10, 50, 90, 99])],
            "first_blocks": tr[:3].tolist(),
        }
        slow = step > 1.5 * med(step)
        if slow.any():
            d["slow_steps"] = int(slow.sum())
            d["slow_team_offchain_done_ns"] = med((rel[:, 10] - done_prev)[slow])
            d["slow_team_read_xprev_ns"] = med((rel[:, 13] - done_prev)[slow])
            d["slow_team_reduced_ns"] = med((rel[:, 0] - done_prev)[slow])
            d["slow_lt_late_landed_ns"] = med((rel[:, 7] - done_prev)[slow])
            d["slow_producer_flag_ns"] = med((rel[:, 5] - done_prev)[slow])
            d["slow_team_q_landed_ns"] = med((rel[:, 6] - done_prev)[slow])
            d["slow_lt_q_sent_ns"] = med((rel[:, 9] - done_prev)[slow])
            d["slow_lt6_q_sent_ns"] = med((rel[:, 2] - done_prev)[slow])
            d["slow_lt_early_done_ns"] = med((rel[:, 11] - done_prev)[slow])
            d["slow_lt_stage_ready_ns"] = med((rel[:, 12] - done_prev)[slow])
            # where the excess goes: steps whose y_k flag came late vs. whose q came late
            late_y = (rel[:, 5] - done_prev) > -500
            late_q = (rel[:, 6] - done_prev) > 350
            d["excess_late_y_us"] = float(ex[late_y].sum() / 1e3)
            d["excess_late_q_not_y_us"] = float(ex[late_q & ~late_y].sum() / 1e3)
        out[nm] = d
    print(json.dumps(out), flush=True)
    s.close()


if __name__ == "__main__":
    main()
