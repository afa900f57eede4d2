#!/usr/bin/env python3
"""Benchmark: BASELINE.json's headline metric on config c2 (1M docs, V=200k, 10k queries, top-10).

One step = one retrieve_batch of the whole 10,000-query batch (doc-tiled scoring + fused
top-k + merge) over an index already resident in HBM. `value` = queries/s from CUDA events
on the library's stream (max over ranks); `e2e` = the same through the public C-ABI call
with pinned HOST buffers (query H2D + result D2H inside the timed region). The index build
(token ids resident on device -> CSC) is reported as index tokens/s beside it.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config 2] [--k 10]
Under torchrun (N>1) the corpus is document-sharded; DF/length statistics are NCCL
all-reduced at build time and per-rank top-k candidates are gathered and merged on rank 0.
`--impl reference` times the CPU port of the reference path (oracle/, all host threads) on
the same config and metric.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "queries/sec (batch, top-10) + index tokens/sec; % of HBM roofline at 1/2/4/8 GPU"
FALLBACK_HBM_GBS = 6650.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "samples": len(sm),
                "reasons": sorted(reasons)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# c3 (BASELINE.json configs[2]) pins delta = 0.5 for BM25L and BM25+; tfldp needs delta > 1/e
VARIANT_DELTA = {"lucene": 0.0, "robertson": 0.0, "atire": 0.0, "bm25l": 0.5, "bm25plus": 0.5, "tfldp": 0.5}


def workload_name(cfg_i, k, variant="lucene"):
    d = VARIANT_DELTA[variant]
    return ({1: "c1", 2: "c2", 3: "c3", 4: "c4", 5: "c5"}[cfg_i] + f" {variant} k1=1.5 b=0.75"
            + (f" delta={d}" if d else "") + f" top-{k}")


# ----------------------------------------------------------------------------- CPU legs
def cpu_corpus(cfg_i):
    from paper_2407_03618_b200 import synth
    cfg = synth.config(cfg_i)
    return synth.corpus_host(cfg, threads=os.cpu_count() or 8)


def cpu_reference_run(cfg_i, k, steps, warmup, sample_q, workers, corp=None, variant="lucene"):
    """Times the CPU port (oracle/) of the reference path: build single-thread, retrieve_batch with `workers`."""
    import oracle
    from paper_2407_03618_b200 import Variant, synth
    corp = corp or cpu_corpus(cfg_i)
    t0 = time.perf_counter()
    ox = oracle.OracleIndex(corp.offsets, corp.tokens, corp.cfg.vocab, int(Variant[variant]), 1.5, 0.75,
                            VARIANT_DELTA[variant])
    build_s = time.perf_counter() - t0
    qoff, qtok = synth.queries(corp.cfg, corp.cdf, 0, sample_q)
    times = []
    for i in range(warmup + steps):
        t = time.perf_counter()
        ids, sc = ox.retrieve_batch(qoff, qtok, k, True, workers)
        if i >= warmup:
            times.append(time.perf_counter() - t)
    qps = sample_q * len(times) / sum(times)
    return {"qps": qps, "build_s": build_s, "tokens": int(corp.offsets[-1]), "ids": ids, "scores": sc,
            "qoff": qoff, "qtok": qtok, "ox": ox, "corp": corp}


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    sample_q = args.ref_sample
    r = cpu_reference_run(args.config, args.k, args.steps, args.warmup, sample_q, cores, variant=args.variant)
    line = {
        "metric": METRIC, "impl": "reference", "value": r["qps"], "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * sample_q / r["qps"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 (oracle accumulator)",
        "data": "synthetic (seeded Zipf corpus/queries, BASELINE.md §5)",
        "config": {"workload": workload_name(args.config, args.k, args.variant), "queries_per_step": sample_q,
                   "k": args.k,
                   "docs": int(len(r["corp"].offsets) - 1), "vocab": int(r["corp"].cfg.vocab)},
        "index_tokens_per_s": r["tokens"] / r["build_s"],
        "cpu_baseline": {"value": r["qps"], "unit": "queries/s", "cores": cores, "kind": "port",
                         "sample": f"{sample_q} queries of c{args.config} per step over the full corpus; "
                                   f"build single-thread {r['build_s']:.1f}s"},
        "e2e": {"value": r["qps"], "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU leg
def text_pipeline_block(cfg_i, hbm, reps=3, cpu_docs=20000):
    """the text side (sl_tokenize, english config: lowercase + bundled
    stopwords + Snowball English) on config c<i>'s corpus rendered as text (synth.render_text).
    Device-resident text timed with CUDA events around the call; e2e from pinned host memory;
    the reference's own tokenizer (oracle/_ref, else the oracle port) on a CPU sample."""
    import torch

    from paper_2407_03618_b200 import synth, text as T
    from paper_2407_03618_b200._lib import SL_MEM_DEVICE, SL_MEM_HOST
    cfg = synth.config(cfg_i)
    corp = synth.corpus_host(cfg, threads=os.cpu_count() or 8)
    words = synth.word_list(cfg.vocab)
    text, off = synth.render_text(corp.tokens, corp.offsets, words, cfg.corpus_seed)
    nb, N = len(text), len(off) - 1
    tc = T.TokenizerConfig.english()
    dtext = torch.from_numpy(text).cuda()
    doff = torch.from_numpy(off.view(np.int64)).cuda()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev_ms, T_out, V = [], 0, 0
    for r in range(reps + 1):
        v = T.Vocabulary()
        torch.cuda.synchronize()
        ev0.record()
        b = T.tokenize_build((dtext, doff), tc, v, mem=SL_MEM_DEVICE)  # the call synchronises its stream
        ev1.record()
        torch.cuda.synchronize()
        if r:
            dev_ms.append(ev0.elapsed_time(ev1))
        T_out, V = b.num_tokens, v.size()
        b.close()
        v.close()
    # e2e through the public streaming call (sl_tokenize_stream): pinned host text in, pinned
    # host (token offsets, ids) out, document-aligned chunks with the copies overlapping the
    # device work; buffers allocated once outside the timed region (a caller reusing them)
    htext = torch.from_numpy(text).pin_memory()
    hoff = torch.from_numpy(off.view(np.int64)).pin_memory()
    h_off = torch.empty(N + 1, dtype=torch.int64).pin_memory()
    h_ids = torch.empty(max(1, T_out), dtype=torch.int32).pin_memory()
    e2e_ms = []
    for r in range(reps + 1):
        v = T.Vocabulary()
        t0 = time.perf_counter()
        _, ids_out = T.tokenize_build_stream(htext, hoff, tc, v, out_ids=h_ids, out_offsets=h_off)
        if r:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        assert ids_out.numel() == T_out
        v.close()
    ms = min(dev_ms)
    alg = nb + 8 * (N + 1) + 4 * T_out + 8 * (N + 1)  # read text + offsets, write ids + token offsets
    ach = alg / (ms / 1e3) / 1e9
    blk = {"workload": f"t{cfg_i}: c{cfg_i} corpus rendered as UTF-8 text (synth.render_text)",
           "tokenizer": "english (lowercase, bundled stopwords, Snowball English)", "docs": N, "bytes": nb,
           "tokens": T_out, "vocab": V, "ms": ms, "bytes_per_s": nb / (ms / 1e3), "tokens_per_s": T_out / (ms / 1e3),
           "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                        "algorithmic_bytes": alg,
                        "note": "per-token string work (raw-string hashing + table probe ~30%, token extraction "
                                "~23%, byte classification ~9%), well below the HBM roofline"},
           "e2e": {"ms": min(e2e_ms), "bytes_per_s": nb / (min(e2e_ms) / 1e3), "h2d_bytes": nb + 8 * (N + 1),
                   "d2h_bytes": 4 * T_out + 8 * (N + 1)}}
    try:
        from oracle.text import TextOracle, ref_available
        kind = "ref" if ref_available() else "port"
        o = TextOracle(kind)
        n = min(N, cpu_docs)
        sample = bytes(text[:int(off[n])])
        t0 = time.perf_counter()
        _, ids, _ = o.tokenize_corpus(sample, off[:n + 1], 1, 1, 1)
        cs = time.perf_counter() - t0
        blk["cpu_baseline"] = {"value": len(sample) / cs, "unit": "bytes/s", "cores": 1,
                               "kind": "reference" if kind == "ref" else "port",
                               "sample": f"first {n} documents ({len(sample)} bytes), tokenize_build, 1 thread",
                               "tokens_per_s": len(ids) / cs}
    except Exception as e:  # noqa: BLE001
        blk["cpu_baseline"] = {"unavailable": str(e)}
    return blk


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2407_03618_b200 import BM25Params, Comm, Variant, _lib, api, build_index, shard_ranges, synth
    from paper_2407_03618_b200._lib import SL_MEM_DEVICE, SL_MEM_HOST, check, lib

    world, rank, local = dist_setup()
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = lib()
    cfg = synth.config(args.config)
    cdf = synth.zipf_cdf(cfg)
    offsets = synth.doc_offsets(cfg)
    if args.shard_of > 1:  # one GPU builds shard `shard_index` of a shard_of-way sharding (c5 memory plan)
        d0, d1 = shard_ranges(offsets, args.shard_of)[args.shard_index]
        # the library caps dense copies by the GLOBAL doc count (12 GB / 4N rows); a shard built
        # with shard-local statistics would not see the full corpus's cap, so pass it explicitly
        os.environ.setdefault("SL_DENSE_MAX_ROWS", str((12 << 30) // (4 * cfg.num_docs)))
    else:
        d0, d1 = shard_ranges(offsets, world)[rank]
    o0, o1 = int(offsets[d0]), int(offsets[d1])
    T_local, T_total = o1 - o0, int(offsets[-1])
    if args.shard_of > 1:
        T_total = T_local
    tok = torch.empty(max(1, T_local), dtype=torch.uint32, device="cuda")
    check(L.sl_synth_tokens_device(cdf.ctypes.data, cfg.vocab, cfg.corpus_seed, o0, T_local, SL_MEM_HOST,
                                   tok.data_ptr()))
    loff = torch.from_numpy((offsets[d0:d1 + 1] - np.uint64(o0)).astype(np.uint64)).cuda()
    comm = None
    if world > 1:
        uid = [Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = Comm(uid[0], world, rank, local)
    params = BM25Params(Variant[args.variant], 1.5, 0.75, VARIANT_DELTA[args.variant])
    # build: warm once (allocator, module load), then the measured build
    idx = build_index(loff, tok, cfg.vocab, params, device=local, doc_base=d0, comm=comm,
                      dense_min_density=args.dense_density)
    idx.close()
    idx = build_index(loff, tok, cfg.vocab, params, device=local, doc_base=d0, comm=comm,
                      dense_min_density=args.dense_density)
    info = idx.info()
    build_ms = torch.tensor([info.build_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(build_ms, op=dist.ReduceOp.MAX)
    build_ms = float(build_ms.item())
    del tok

    qoff, qtok = synth.queries(cfg, cdf)
    B, k = len(qoff) - 1, args.k
    d_off = torch.from_numpy(qoff.astype(np.uint64)).cuda()
    d_tok = torch.from_numpy(qtok.astype(np.uint32)).cuda()
    ids = torch.empty((B, k), dtype=torch.uint32, device="cuda")
    scs = torch.empty((B, k), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    st = _lib.RetrieveStats()

    def step_device():
        check(L.sl_retrieve_batch_timed(idx.handle, d_off.data_ptr(), d_tok.data_ptr(), B, k, SL_MEM_DEVICE,
                                        ids.data_ptr() if rank == 0 else None,
                                        scs.data_ptr() if rank == 0 else None, C.byref(st)))
        return st.total_ms, st.score_kernel_ms, st.posting_bytes, st.scorevec_bytes, st.kernels_launched

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step_device()
    tot_ms, ker_ms, launches = 0.0, 0.0, 0
    pb = sb = 0
    barrier()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (256 MiB > 126 MB L2), outside the events
            torch.cuda.synchronize()
            a, b, pb, sb, nl = step_device()
            tot_ms += a
            ker_ms += b
            launches += nl
        barrier()
    clocks = clk.summary()
    t = torch.tensor([tot_ms, ker_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms, ker_ms = float(t[0]), float(t[1])
    res_ids = ids.cpu().numpy() if rank == 0 else None

    # e2e through the public C-ABI with pinned host buffers (H2D queries + D2H results in the region)
    h_off = torch.from_numpy(qoff.astype(np.uint64)).pin_memory()
    h_tok = torch.from_numpy(qtok.astype(np.uint32)).pin_memory()
    h_ids = torch.empty((B, k), dtype=torch.uint32).pin_memory()
    h_sc = torch.empty((B, k), dtype=torch.float32).pin_memory()
    for _ in range(args.warmup):
        check(L.sl_retrieve_batch(idx.handle, h_off.data_ptr(), h_tok.data_ptr(), B, k, 1, SL_MEM_HOST,
                                  h_ids.data_ptr(), h_sc.data_ptr()))
    barrier()
    e2e_s = 0.0
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        t0 = time.perf_counter()
        check(L.sl_retrieve_batch(idx.handle, h_off.data_ptr(), h_tok.data_ptr(), B, k, 1, SL_MEM_HOST,
                                  h_ids.data_ptr(), h_sc.data_ptr()))
        barrier()
        e2e_s += time.perf_counter() - t0
    e2e = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e.item())

    if rank == 0:
        hbm, hbm_src = peaks()
        bytes_per_launch = pb + sb
        achieved = bytes_per_launch / (ker_ms / args.steps / 1e3) / 1e9
        # unique posting bytes of the batch (cross-query reuse potential), from the exported indptr
        V = cfg.vocab
        indptr = np.empty(V + 1, np.uint64)
        check(L.sl_index_export(idx.handle, SL_MEM_HOST, indptr.ctypes.data, None, None, None, None, None, None))
        nnz_t = np.diff(indptr.astype(np.int64))
        uniq = 8 * int(nnz_t[np.unique(qtok)].sum()) + 4 * info.num_docs_local * B
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(f"c{args.config}_k{k}_per_launch")
        qps = B * args.steps / (tot_ms / 1e3)
        line = {
            "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 accumulate (f64 build math)",
            "data": "synthetic (seeded Zipf corpus/queries, BASELINE.md §5; BEIR absent)",
            "config": {"workload": workload_name(args.config, k, args.variant), "docs": cfg.num_docs,
                       "vocab": cfg.vocab,
                       "tokens": T_total, "nnz_local": int(info.nnz_local), "queries_per_step": B, "k": k,
                       "parallelism": f"doc-shard x{world}", "l2": "flushed between steps (256 MiB memset)",
                       "dense_rows": int(info.dense_rows), "skip_rows": int(info.skip_rows),
                       "tile_docs": int(info.tile_docs),
                       **({"simulated_shard": f"{args.shard_index} of {args.shard_of} (docs {d0}..{d1}; "
                                              "shard-local df/N statistics; value is per-GPU)"}
                          if args.shard_of > 1 else {})},
            "index_tokens_per_s": T_total / (build_ms / 1e3),
            "index_build": {
                "ms": build_ms, "tokens": T_total, "nnz": int(info.nnz_local),
                # SURVEY §8d floor: read ids + offsets, write CSC, indptr, doclens, df, theta
                "algorithmic_bytes": 4 * T_total + 8 * (int(info.num_docs_local) + 1) + 8 * int(info.nnz_local)
                                     + 8 * (cfg.vocab + 1) + 4 * int(info.num_docs_local) + 8 * cfg.vocab,
            },
            "score_kernel_ms_per_step": ker_ms / args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "peak_source": hbm_src, "traffic": traffic,
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "posting_bytes_per_launch": pb, "scorevec_bytes_per_launch": sb,
                         "unique_bytes_per_launch": uniq,
                         "note": "per-query posting+score-vector bytes, no cross-query dedup (SURVEY §8d); "
                                 "frac > 1 comes from cross-query reuse (shared dense head rows in L2)"},
            "e2e": {"value": B * args.steps / e2e_s, "unit": "queries/s",
                    "h2d_bytes_per_step": int(h_off.numel() * 8 + h_tok.numel() * 4),
                    "d2h_bytes_per_step": int(B * k * 8)},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        bb = line["index_build"]["algorithmic_bytes"]
        line["index_build"]["achieved_GBps"] = bb / (build_ms / 1e3) / 1e9
        line["index_build"]["frac"] = line["index_build"]["achieved_GBps"] / hbm
        if world == 1 and not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            r = cpu_reference_run(args.config, k, 1, 1, args.cpu_sample, cores, variant=args.variant)
            line["cpu_baseline"] = {"value": r["qps"], "unit": "queries/s", "cores": cores, "kind": "port",
                                    "sample": f"first {args.cpu_sample} queries of c{args.config}, full 1M-doc "
                                              f"index; CPU build (1 thread) {r['build_s']:.1f}s = "
                                              f"{r['tokens'] / r['build_s']:.3g} tokens/s"}
            agree = float(np.mean(res_ids[: args.cpu_sample] == r["ids"]))
            line["parity_sample"] = {"queries": args.cpu_sample, "top_k_id_agreement": agree}
        if world == 1 and not args.no_text:
            line["text_pipeline"] = text_pipeline_block(args.config, hbm)
        print(json.dumps(line), flush=True)
    idx.close()
    if comm:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--variant", choices=list(VARIANT_DELTA), default="lucene",
                    help="BM25 variant (c3 sweeps robertson, atire, bm25l, bm25plus on c2's corpus)")
    ap.add_argument("--dense-density", type=float, default=0.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-text", action="store_true", help="skip the text-pipeline block")
    ap.add_argument("--cpu-sample", type=int, default=64)
    ap.add_argument("--ref-sample", type=int, default=128)
    ap.add_argument("--shard-of", type=int, default=1, help="build one shard of an N-way doc sharding (1 GPU)")
    ap.add_argument("--shard-index", type=int, default=0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    return run_reference(args) if args.impl == "reference" else run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
