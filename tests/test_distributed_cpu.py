"""Multi-rank host protocol of the document-sharded path, on CPU with gloo (world_size 2).

The GPU path runs exactly this protocol with NCCL inside libsparselex_b200:
contiguous doc ranges balanced by tokens (shard_ranges), all-reduce of df / N / Σ|D|,
per-shard build with the global statistics, per-shard top-k with global doc ids, gather to
rank 0 and a (score desc, doc asc) merge. Here the per-shard compute is the CPU oracle and
the exchange is torch.distributed gloo; the merged result must equal the unsharded oracle.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out_dir):
    import oracle
    from paper_2407_03618_b200 import shard_ranges, synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    cfg = synth.config(1, num_docs=4000)
    corp = synth.corpus_host(cfg, threads=2)
    qoff, qtok = synth.queries(cfg, corp.cdf, 0, 200)
    d0, d1 = shard_ranges(corp.offsets, WORLD)[rank]
    o0 = int(corp.offsets[d0])
    off = (corp.offsets[d0:d1 + 1] - np.uint64(o0)).astype(np.uint64)
    tok = corp.tokens[o0:int(corp.offsets[d1])]
    for variant, delta in [(2, 0.0), (4, 0.5), (0, 0.0)]:
        local = oracle.OracleIndex(off, tok, cfg.vocab, variant, 1.5, 0.75, delta)
        df = torch.from_numpy(local.export()["df"].astype(np.int64))
        st = torch.tensor([int(off[-1]), d1 - d0], dtype=torch.int64)
        dist.all_reduce(df)  # C1
        dist.all_reduce(st)  # C2
        shard = oracle.OracleIndex(off, tok, cfg.vocab, variant, 1.5, 0.75, delta,
                                   global_stats=(df.numpy().astype(np.uint32), int(st[1]), int(st[0])))
        k = 10
        ids, sc = shard.retrieve_batch(qoff, qtok, k, True, 2)
        ids = np.where(ids == 0xFFFFFFFF, ids, ids + np.uint32(d0))  # global doc ids
        gi = [torch.zeros(ids.shape, dtype=torch.int64) for _ in range(WORLD)]
        gs = [torch.zeros(sc.shape, dtype=torch.float64) for _ in range(WORLD)]
        dist.all_gather(gi, torch.from_numpy(ids.astype(np.int64)))  # C3 (gather to rank 0)
        dist.all_gather(gs, torch.from_numpy(sc))
        if rank == 0:
            full = oracle.OracleIndex(corp.offsets, corp.tokens, cfg.vocab, variant, 1.5, 0.75, delta)
            rid, rsc = full.retrieve_batch(qoff, qtok, k, True, 2)
            for b in range(len(qoff) - 1):
                c = [(float(gs[r][b, j]), int(gi[r][b, j])) for r in range(WORLD) for j in range(k)
                     if gi[r][b, j] != 0xFFFFFFFF]
                c.sort(key=lambda x: (-x[0], x[1]))  # K7 merge
                assert [i for _, i in c[:k]] == rid[b].tolist(), (variant, b)
                assert [s for s, _ in c[:k]] == rsc[b].tolist(), (variant, b)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        open(os.path.join(out_dir, "ok"), "w").write("ok")


def test_sharded_protocol_gloo(tmp_path):
    mp.spawn(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    assert (tmp_path / "ok").exists()


def test_shard_ranges_balance_tokens():
    from paper_2407_03618_b200 import shard_ranges
    off = np.concatenate([[0], np.cumsum(np.r_[np.full(100, 10), np.full(10, 1000)])]).astype(np.uint64)
    r = shard_ranges(off, 4)
    assert r[0][0] == 0 and r[-1][1] == 110
    assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
