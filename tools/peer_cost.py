"""Cost of the fused peer combine on one GPU (GPU box): the sharded asum /
dot kernel timed like bench.py with and without the in-kernel exchange
(world = 1, so the rank publishes to and waits on its own mailbox; across
GPUs the same code adds one NVLink store per peer and the wait for the
slowest rank).  Measurement infrastructure only.

    python tools/peer_cost.py
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.scaleout import ShardedReduction  # noqa: E402


def main():
    RT.init(0)
    st = RT.Stream(0)
    for kind, total in (("asum", 1 << 28), ("asum", 1 << 26), ("dot", 1 << 25)):
        res = {}
        for combine in ("nccl", "peer"):
            run = ShardedReduction(kind, total, combine=combine)
            run.fill_inputs(st)
            ts = []
            for i in range(45):
                RT.lib().dpia_l2_flush(0, st.handle)
                e0, e1 = RT.Event(0), RT.Event(0)
                e0.record(st)
                run.launch(st, allreduce=False)
                e1.record(st)
                st.sync()
                if i >= 5:
                    ts.append(e0.elapsed_ms(e1))
            res[combine] = (statistics.mean(ts) * 1e3, run.result())
            if run.peer is not None:
                run.peer.check()
                run.peer.close()
        print(f"{kind} 2^{total.bit_length() - 1}: no combine {res['nccl'][0]:.2f} us, fused peer combine "
              f"{res['peer'][0]:.2f} us (+{res['peer'][0] - res['nccl'][0]:.2f} us); results equal: "
              f"{res['nccl'][1] == res['peer'][1]}", flush=True)


if __name__ == "__main__":
    main()
