"""Run tests/test_sharded.py's world-2 sbbf_dist hooks worker standalone with
stack dumps on a hang (debug aid)."""
import faulthandler
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch.multiprocessing as mp  # noqa: E402


def worker(rank, world, port, total, q):
    faulthandler.enable(file=sys.stderr)
    faulthandler.dump_traceback_later(45, exit=True, file=sys.stderr)
    from tests import test_sharded as T
    print(f"rank {rank} start", file=sys.stderr, flush=True)
    T._dist_hooks_worker(rank, world, port, total, q)
    print(f"rank {rank} done", file=sys.stderr, flush=True)


if __name__ == "__main__":
    from tests.test_sharded import free_port
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker, args=(r, 2, port, 1 << 20, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        print("exitcode", p.exitcode, flush=True)
    while not q.empty():
        g = q.get()
        print("got", g[0], g[1] if isinstance(g[1], str) else "ok", g[2] if isinstance(g[1], str) else "")
