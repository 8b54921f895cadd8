"""Multi-GPU host logic on CPU: gloo, world_size 2 (no GPU needed).

The 8-GPU path is: interleaved blocks per rank (wv_shard_blocks,
the same partition wv_search_shard sieves), independent compute, then an
all_gather of counts / hit lists / checksums and a sorted merge
(paper_2101_11157_b200.dist.gather_results).  Here each rank fills its shard's
result arrays from the CPU oracle's prime list (residue values are stand-ins:
this test checks the partition and the collective merge, not arithmetic), and
the merged result must equal the single-process one byte for byte.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

LO, HI, BLOCK = 1000, 1000 + 11 * 131072 + 4321, 131072


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_arrays(wv, oracle, lo, hi, shard, nshards, block):
    blocks, used = wv.shard_blocks(lo, hi, shard, nshards, block)
    ps = []
    for a, b in blocks:
        ps += oracle.primes(max(a, 5), b)
    res = np.zeros(len(ps), dtype=wv.RES_DTYPE)
    res["p"] = ps
    res["res_w"] = [p % 1009 for p in ps]
    res["res_v"] = [(p * 7) % 997 for p in ps]
    flags = (res["res_w"] == 0).astype(np.uint32) | 2 * (res["res_v"] == 0).astype(np.uint32)
    hits = np.zeros(int((flags > 0).sum()), dtype=wv.HIT_DTYPE)
    hits["p"] = res["p"][flags > 0]
    hits["flags"] = flags[flags > 0]
    chk = 0
    for r in res:
        chk = (chk + wv.checksum_term(int(r["p"]), int(r["res_w"]), int(r["res_v"]))) % (1 << 64)
    return hits, res, chk, blocks


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2101_11157_b200 as wv
    from paper_2101_11157_b200.dist import gather_results
    hits, res, chk, blocks = _local_arrays(wv, oracle, LO, HI, rank, world, BLOCK)
    h, r, c = gather_results(hits, res, chk)
    out_q.put((rank, h.tobytes(), r.tobytes(), c, blocks))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_gather_equals_single_process(world):
    import oracle
    import paper_2101_11157_b200 as wv
    import __graft_entry__ as g
    g.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    h1, r1, c1, _ = _local_arrays(wv, oracle, LO, HI, 0, 1, BLOCK)
    blocks_all = []
    for rank, hb, rb, c, blocks in outs:
        assert hb == h1.tobytes() and rb == r1.tobytes() and c == c1, rank
        blocks_all += blocks
    # the shards' blocks tile [LO, HI) exactly, interleaved
    blocks_all.sort()
    assert blocks_all[0][0] == LO and blocks_all[-1][1] == HI
    assert all(a[1] == b[0] for a, b in zip(blocks_all, blocks_all[1:]))
    mine = {rank: blocks for rank, _, _, _, blocks in outs}
    assert mine[0][0][0] == LO and mine[1][0][0] == LO + BLOCK
    # snake interleave: round 1 is dealt in reverse (block 2 -> rank 1, block 3 -> rank 0)
    assert mine[1][1][0] == LO + 2 * BLOCK and mine[0][1][0] == LO + 3 * BLOCK


def test_shard_blocks_default_block_sizes():
    import paper_2101_11157_b200 as wv
    import __graft_entry__ as g
    g.build()
    # C5 over 8 shards: >= 32 blocks per shard
    b, used = wv.shard_blocks(39 * 10 ** 9, 40 * 10 ** 9, 3, 8)
    assert used == 1 << 21 and len(b) >= 32
    # unsharded: one block covering the window
    b, used = wv.shard_blocks(5, 3 * 10 ** 6, 0, 1)
    assert b == [(5, 3 * 10 ** 6)]
    with pytest.raises(wv.WVError):
        wv.shard_blocks(5, 100, 2, 2)
    with pytest.raises(wv.WVError):
        wv.shard_blocks(5, 10 ** 6, 0, 2, 1000)     # block not a multiple of the sieve span
