"""Multi-rank path on CPU (gloo, world_size 2): frame-range shards partition
the global frame set, and the counters reduced across ranks equal a single
process's counters on the same frames (the multi-GPU analogue of
test_sim.cpp:37-66 worker-count independence).  The per-rank decode here is
the C oracle (CPU); on GPUs bench.py runs the same logic with the sm_100a
decoder and NCCL."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _decode_counts(lo, hi):
    sys.path.insert(0, ROOT)
    import paper_1710_08314_b200 as P
    from oracle.oracle import Oracle
    from paper_1710_08314_b200.shard import Counters

    code = P.make_code(128, 48, P.construct_frozen(128, 56, 0.5), "8")
    info, llr = P.channel(code, 1.5, 42, lo, hi - lo, "f32", nthreads=1)
    c = code.crc
    o = Oracle(128, 48, code.frozen, (c.width, c.poly, int(c.reflect), c.init, c.xorout),
               "fa_sscl", 8, "f32").decode(llr)
    cnt = Counters()
    cnt.add_batch(np.unpackbits(o.payload, axis=1), info, o.esc)
    return cnt


def _worker(rank, world, port, frames_per_rank, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_1710_08314_b200.shard import all_reduce_counters, frame_range

    lo, hi = frame_range(rank, world, frames_per_rank)
    tot = all_reduce_counters(_decode_counts(lo, hi))
    q.put((rank, lo, hi, tot.as_array().tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_frame_ranges_partition():
    sys.path.insert(0, ROOT)
    from paper_1710_08314_b200.shard import frame_range, split_range

    for world in (1, 2, 4, 8):
        got = [frame_range(r, world, 100, 7) for r in range(world)]
        assert got[0][0] == 7 and all(got[i][1] == got[i + 1][0] for i in range(world - 1))
        sp = [split_range(r, world, 1001) for r in range(world)]
        assert sp[0][0] == 0 and sp[-1][1] == 1001 and sum(b - a for a, b in sp) == 1001


def test_two_rank_counters_equal_single_process():
    world, fpr = 2, 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fpr, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    res.sort()
    assert [(a, b) for _, a, b, _ in res] == [(0, fpr), (fpr, 2 * fpr)]
    assert res[0][3] == res[1][3]  # every rank holds the reduced totals
    single = _decode_counts(0, world * fpr).as_array().tolist()
    assert res[0][3] == single
    assert single[0] == world * fpr and single[2] > 0  # some frame errors at 1.5 dB
