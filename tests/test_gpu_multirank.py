"""The multi-rank protocol on the real CUDA path: two processes on one GPU, gloo in between.

NCCL cannot put two ranks on one device, and gpurun gives one GPU, so the library's own
NCCL exchange (sl_comm) is covered with one rank in test_gpu_sharding.py. Here the SAME
protocol steps run through libsparselex_b200 in two processes, with torch.distributed gloo as
the transport:
  C1/C2  each rank builds its token-balanced shard, exports its df, and the df / N / Σ|D|
         are all-reduced over gloo; each rank rebuilds with the corpus-wide statistics
         (sl_build_desc.global_df -- the path a caller with its own transport uses);
  K5/K6  sl_retrieve_local: per-rank top-k candidate keys with global doc ids;
  C3/K7  the keys are gathered to rank 0 and merged by sl_merge_candidates.
Rank 0's merged (ids, scores) must be BIT-IDENTICAL to retrieve_batch on the unsharded index,
with and without query-batch chunking (SL_CAND_MB=1 forces many chunks).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out_dir, cand_mb):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if cand_mb:
        os.environ["SL_CAND_MB"] = str(cand_mb)
    from paper_2407_03618_b200 import (BM25Params, Variant, build_index, merge_candidates, retrieve_batch,
                                       retrieve_local, shard_ranges, synth)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    cfg = synth.config(1, num_docs=20000)
    corp = synth.corpus_host(cfg, threads=4)
    qoff, qtok = synth.queries(cfg, corp.cdf, 0, 600)
    d0, d1 = shard_ranges(corp.offsets, WORLD)[rank]
    o0 = int(corp.offsets[d0])
    off = (corp.offsets[d0:d1 + 1] - np.uint64(o0)).astype(np.uint64)
    tok = corp.tokens[o0:int(corp.offsets[d1])]
    for p in (BM25Params(Variant.lucene), BM25Params(Variant.bm25plus, 1.5, 0.75, 0.5),
              BM25Params(Variant.robertson)):
        with build_index(off, tok, cfg.vocab, p, device=0) as local:
            df = torch.from_numpy(local.export()["df"].astype(np.int64))
        st = torch.tensor([int(off[-1]), d1 - d0], dtype=torch.int64)
        dist.all_reduce(df)  # C1
        dist.all_reduce(st)  # C2
        gstats = (df.numpy().astype(np.uint32), int(st[1]), int(st[0]))
        with build_index(off, tok, cfg.vocab, p, device=0, doc_base=d0, global_stats=gstats) as shard:
            assert shard.num_docs == cfg.num_docs
            ex = shard.export()
            for k in (10, 100):
                keys, qc = retrieve_local(shard, (qoff, qtok), k)
                kt = torch.from_numpy(keys.view(np.int64))
                parts = [torch.zeros_like(kt) for _ in range(WORLD)]
                dist.all_gather(parts, kt)  # C3 (rank 0 uses every part)
                qcs = [torch.zeros(len(qc), dtype=torch.float64) for _ in range(WORLD)]
                dist.all_gather(qcs, torch.from_numpy(qc))
                if rank == 0:
                    for q in qcs[1:]:  # the query constant is a global quantity
                        assert torch.equal(q, qcs[0])
                    allk = np.stack([t.numpy().view(np.uint64) for t in parts])
                    ids, sc = merge_candidates(allk, qc)  # K7
                    with build_index(corp.offsets, corp.tokens, cfg.vocab, p, device=0) as full:
                        if k == 10:
                            fx = full.export()
                            np.testing.assert_array_equal(fx["df"], ex["df"])
                            assert fx["avg_len"] == ex["avg_len"]
                        rid, rsc = retrieve_batch(full, (qoff, qtok), k, as_arrays=True)
                    np.testing.assert_array_equal(sc, rsc, err_msg=f"{p.variant.name} k={k}")
                    np.testing.assert_array_equal(ids, rid, err_msg=f"{p.variant.name} k={k}")
                dist.barrier()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        open(os.path.join(out_dir, "ok"), "w").write("ok")


@pytest.mark.parametrize("cand_mb", [0, 1], ids=["one-chunk", "chunked"])
def test_two_ranks_one_gpu_bit_identical(cuda_ok, tmp_path, cand_mb):
    mp.spawn(_worker, args=(_free_port(), str(tmp_path), cand_mb), nprocs=WORLD, join=True)
    assert (tmp_path / "ok").exists()
