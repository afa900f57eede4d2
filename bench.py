#!/usr/bin/env python3
"""Benchmark: BASELINE.json's headline metric on config c2 (1M docs, V=200k, 10k queries, top-10).

One step = one retrieve_batch of the whole 10,000-query batch (doc-tiled scoring + fused
top-k + merge) over an index already resident in HBM. `value` = queries/s from CUDA events
on the library's stream (max over ranks); `e2e` = the same through the public C-ABI call
with pinned HOST buffers (query H2D + result D2H inside the timed region). The index build
(token ids resident on device -> CSC) is reported as index tokens/s beside it.
`roofline` carries the scoring kernel's PHYSICAL DRAM traffic, issue and L2 fractions, taken
in this run by an ncu child process over one launch of the same batch (ncu_probe); the SURVEY
§8d algorithmic bytes (no cross-query dedup) appear as `reuse_factor`.
More blocks of the same line: c2 top-100, the c3 variant sweep (Robertson, ATIRE, BM25L, BM25+),
c4 top-1000 (every N), c5 top-100 (N = 8), the CPU baseline (single-thread and all cores,
host model / RAM) and the text pipeline.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config 2] [--k 10]
Under torchrun (N>1) the corpus is document-sharded; DF/length statistics are NCCL
all-reduced at build time and per-rank top-k candidates are gathered and merged on rank 0
(NCCL_DEBUG=INFO / SUBSYS=INIT shows the communicator's nranks).
`--impl reference` times the CPU port of the reference path (oracle/, all host threads) on
the same config (the whole 10k-query batch per step) and metric.
"""
from __future__ import annotations

import argparse
import csv
import ctypes as C
import json
import os
import shutil
import subprocess
import sys
import tempfile
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


# ----------------------------------------------------------------------------- host / config
def host_info():
    """CPU model, logical CPUs and RAM of the box the CPU legs run on (SPEC cmd_bench context)."""
    model, ram_gb = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram_gb = round(int(line.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    return {"cpu": model, "logical_cpus": os.cpu_count(), "ram_gb": ram_gb}


def bench_config(cfg_i, k, variant, docs, vocab, tokens, queries_per_step):
    """The workload both arms print (identical dicts: the driver's same_config check)."""
    return {"workload": workload_name(cfg_i, k, variant), "docs": int(docs), "vocab": int(vocab),
            "tokens": int(tokens), "queries_per_step": int(queries_per_step), "k": int(k)}


# ----------------------------------------------------------------------------- CPU legs
def cpu_corpus(cfg_i):
    from paper_2407_03618_b200 import synth
    cfg = synth.config(cfg_i)
    return synth.corpus_host(cfg, threads=os.cpu_count() or 8)


def cpu_index(corp, variant):
    """The CPU port (oracle/) of the reference's two-pass build_index, single-threaded (timed)."""
    import oracle
    from paper_2407_03618_b200 import Variant
    t0 = time.perf_counter()
    ox = oracle.OracleIndex(corp.offsets, corp.tokens, corp.cfg.vocab, int(Variant[variant]), 1.5, 0.75,
                            VARIANT_DELTA[variant])
    return ox, time.perf_counter() - t0


def cpu_qps(ox, qoff, qtok, nq, k, workers, reps=1):
    """retrieve_batch of the first nq queries with `workers` threads: (QPS, ids of the last rep)."""
    off, tok = qoff[:nq + 1], qtok[:int(qoff[nq])]
    t = 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        ids, _ = ox.retrieve_batch(off, tok, k, True, workers)
        t += time.perf_counter() - t0
    return nq * reps / t, ids


def run_reference(args):
    """The reference arm: the CPU port of the reference path on this box's host cores, the same
    config / metric as our arm (the full query batch per step, all host threads: SPEC
    retrieve_batch `workers`), plus the single-thread QPS (the paper's methodology) on a sample."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return 0
    from paper_2407_03618_b200 import synth
    cores = os.cpu_count() or 1
    corp = cpu_corpus(args.config)
    ox, build_s = cpu_index(corp, args.variant)
    qoff, qtok = synth.queries(corp.cfg, corp.cdf)
    B = len(qoff) - 1 if args.ref_sample <= 0 else min(args.ref_sample, len(qoff) - 1)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ox.retrieve_batch(qoff[:B + 1], qtok[:int(qoff[B])], args.k, True, cores)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    qps = B * len(times) / sum(times)
    n1 = min(B, args.cpu_sample)
    qps1, _ = cpu_qps(ox, qoff, qtok, n1, args.k, 1)
    T = int(corp.offsets[-1])
    line = {
        "metric": METRIC, "impl": "reference", "value": qps, "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 (oracle accumulator)",
        "data": "synthetic (seeded Zipf corpus/queries, BASELINE.md §5)",
        "config": bench_config(args.config, args.k, args.variant, corp.cfg.num_docs, corp.cfg.vocab, T, B),
        "parallelism": f"CPU, {cores} worker threads (SPEC retrieve_batch workers)",
        "index_tokens_per_s": T / build_s,
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": cores, "kind": "port",
                         "sample": f"all {B} queries of c{args.config} per step over the full corpus; "
                                   f"build single-thread {build_s:.1f}s",
                         "single_thread": {"value": qps1, "unit": "queries/s", "cores": 1,
                                           "sample": f"first {n1} queries, workers=1"},
                         "host": host_info()},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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


# ----------------------------------------------------------------------------- physical counters
NCU_METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum",
               "smsp__issue_active.avg.pct_of_peak_sustained_active",
               "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
               "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]


def ncu_probe(cfg_i, k, variant, dense_density, timeout=300):
    """Physical counters of the scoring kernel IN THIS RUN: ncu over a child process that builds
    the same index and runs one retrieve_batch of the same batch (one k_score_runs launch, L2
    cold as in the flushed timed steps). The child's timings are never bench values; only its
    DRAM / L2 / issue counters are used."""
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return {"error": "ncu not found"}
    cmd = [ncu, "--metrics", ",".join(NCU_METRICS), "--clock-control", "none", "-k", "regex:k_score_runs", "-c", "1",
           "--csv", sys.executable, os.path.abspath(__file__), "--ncu-child", "--config", str(cfg_i), "--k", str(k),
           "--variant", variant, "--dense-density", str(dense_density)]
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    t0 = time.perf_counter()
    try:
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    except subprocess.TimeoutExpired:
        return {"error": f"ncu timed out after {timeout}s"}
    vals = {}
    rows = list(csv.reader(ln for ln in p.stdout.splitlines() if ln.startswith('"')))
    if rows:
        hdr = rows[0]
        try:
            ni, vi = hdr.index("Metric Name"), hdr.index("Metric Value")
            for r in rows[1:]:
                vals[r[ni]] = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            pass
    if "dram__bytes_read.sum" not in vals:
        return {"error": f"ncu rc={p.returncode}: {(p.stderr or p.stdout)[-300:]}"}
    vals["probe_s"] = time.perf_counter() - t0
    return vals


def physical_roofline(ncu, kernel_ms, alg_bytes, uniq_bytes, hbm, hbm_src, sms):
    """roofline block: DRAM bytes the scoring kernel moved (ncu, this run) / its live time / peak,
    the SURVEY §8d algorithmic bytes kept as a reuse factor, issue and L2 fractions."""
    if "error" in ncu:
        return {"bound": "hbm", "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None, "traffic": None,
                "traffic_error": ncu["error"], "algorithmic_bytes_per_launch": alg_bytes,
                "unique_bytes_per_launch": uniq_bytes, "peak_source": hbm_src}
    dram = ncu["dram__bytes_read.sum"] + ncu["dram__bytes_write.sum"]
    ach = dram / (kernel_ms / 1e3) / 1e9
    t_ncu = ncu["gpu__time_duration.sum"] * 1e-9
    clk = ncu.get("sm__cycles_elapsed.avg.per_second", 0.0)
    issue = ncu["smsp__inst_executed.sum"] / (4 * sms * clk * t_ncu) if clk and t_ncu else None
    return {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": dram,
            "peak_source": hbm_src,
            "measured": "DRAM read+write bytes of one k_score_runs launch (ncu child of this run, same index and "
                        "batch, L2 cold) over the live kernel time (CUDA events, this run)",
            "kernel_ms": kernel_ms, "ncu_kernel_ms": t_ncu * 1e3,
            "algorithmic_bytes_per_launch": alg_bytes, "unique_bytes_per_launch": uniq_bytes,
            "reuse_factor": alg_bytes / dram,
            "issue_frac": issue,
            "issue_active_frac": ncu["smsp__issue_active.avg.pct_of_peak_sustained_active"] / 100,
            "l2_frac": ncu["lts__t_sectors.avg.pct_of_peak_sustained_elapsed"] / 100,
            "l2_bytes": ncu["lts__t_bytes.sum"],
            "l1_frac": ncu["l1tex__throughput.avg.pct_of_peak_sustained_active"] / 100,
            "binding_limit": "instruction issue and L2 latency, not HBM: the batch's posting and score bytes "
                             "(algorithmic, SURVEY §8d, no cross-query dedup) are served from L2 / shared memory "
                             "reuse_factor times over"}


# ----------------------------------------------------------------------------- GPU leg
class Shard:
    """This rank's index shard of config c<cfg_i> (token-balanced contiguous doc range), built
    twice (warm-up, then measured) from device-generated tokens."""

    def __init__(self, cfg_i, variant, world, rank, local, comm, dense_density, shard_of=1, shard_index=0):
        import torch
        import torch.distributed as dist
        from paper_2407_03618_b200 import BM25Params, Variant, build_index, shard_ranges, synth
        self.cfg = cfg = synth.config(cfg_i)
        self.cdf = cdf = synth.zipf_cdf(cfg)
        offsets = synth.doc_offsets(cfg)
        if shard_of > 1:  # one GPU builds one shard of a shard_of-way sharding (shard-local statistics)
            d0, d1 = shard_ranges(offsets, shard_of)[shard_index]
            os.environ.setdefault("SL_DENSE_MAX_ROWS", str((12 << 30) // (4 * cfg.num_docs)))
        else:
            d0, d1 = shard_ranges(offsets, world)[rank]
        o0, o1 = int(offsets[d0]), int(offsets[d1])
        self.d0, self.d1 = d0, d1
        self.T_local = o1 - o0
        self.T_total = self.T_local if shard_of > 1 else int(offsets[-1])
        tok = torch.empty(max(1, self.T_local), dtype=torch.uint32, device="cuda")
        synth.tokens_device(cfg, cdf, o0, self.T_local, tok.data_ptr())
        loff = torch.from_numpy((offsets[d0:d1 + 1] - np.uint64(o0)).astype(np.uint64)).cuda()
        p = BM25Params(Variant[variant], 1.5, 0.75, VARIANT_DELTA[variant])
        idx = build_index(loff, tok, cfg.vocab, p, device=local, doc_base=d0, comm=comm,
                          dense_min_density=dense_density)
        idx.close()
        self.idx = build_index(loff, tok, cfg.vocab, p, device=local, doc_base=d0, comm=comm,
                               dense_min_density=dense_density)
        self.info = self.idx.info()
        bm = torch.tensor([self.info.build_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(bm, op=dist.ReduceOp.MAX)
        self.build_ms = float(bm.item())
        del tok, loff
        torch.cuda.empty_cache()

    def build_block(self, hbm):
        inf, V = self.info, self.cfg.vocab
        # SURVEY §8d floor: read ids + offsets, write CSC, indptr, doclens, df, theta (this rank)
        alg = (4 * self.T_local + 8 * (inf.num_docs_local + 1) + 8 * inf.nnz_local + 8 * (V + 1)
               + 4 * inf.num_docs_local + 8 * V)
        return {"ms": self.build_ms, "tokens": self.T_total, "tokens_per_s": self.T_total / (self.build_ms / 1e3),
                "nnz_local": int(inf.nnz_local), "algorithmic_bytes_rank": alg,
                "achieved_GBps_rank": alg / (self.build_ms / 1e3) / 1e9,
                "frac": alg / (self.build_ms / 1e3) / 1e9 / hbm,
                "index": {"dense_rows": int(inf.dense_rows), "skip_rows": int(inf.skip_rows),
                          "tile_docs": int(inf.tile_docs), "device_bytes": int(inf.device_bytes)}}

    def close(self):
        self.idx.close()


def time_retrieval(L, idx, qoff, qtok, k, steps, warmup, rank, world, flush, clock_dev=None, e2e=True):
    """Device-timed retrieve_batch over the whole batch (sl_retrieve_batch_timed, CUDA events on
    the library's stream, L2 flushed before each step, max over ranks) and, optionally, the
    same through the public call with pinned host buffers (e2e, wall clock, max over ranks)."""
    import torch
    import torch.distributed as dist
    from paper_2407_03618_b200 import _lib
    from paper_2407_03618_b200._lib import SL_MEM_DEVICE, SL_MEM_HOST, check
    B = len(qoff) - 1
    d_off = torch.from_numpy(qoff.astype(np.uint64)).cuda()
    d_tok = torch.from_numpy(qtok.astype(np.uint32)).cuda()
    ids = torch.empty((B, k), dtype=torch.uint32, device="cuda")
    scs = torch.empty((B, k), dtype=torch.float32, device="cuda")
    st = _lib.RetrieveStats()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        check(L.sl_retrieve_batch_timed(idx.handle, d_off.data_ptr(), d_tok.data_ptr(), B, k, SL_MEM_DEVICE,
                                        ids.data_ptr() if rank == 0 else None, scs.data_ptr() if rank == 0 else None,
                                        C.byref(st)))
        return st.total_ms, st.score_kernel_ms, st.merge_ms, st.posting_bytes, st.scorevec_bytes, st.kernels_launched

    for _ in range(warmup):
        step()
    tot = ker = mrg = 0.0
    launches = pb = sb = 0
    barrier()
    clk = ClockSampler(clock_dev) if clock_dev is not None else None
    if clk:
        clk.__enter__()
    for _ in range(steps):
        flush.zero_()  # L2 flush between timed steps (256 MiB > 126 MB L2), outside the events
        torch.cuda.synchronize()
        a, b, c, pb, sb, nl = step()
        tot, ker, mrg, launches = tot + a, ker + b, mrg + c, launches + nl
    barrier()
    if clk:
        clk.__exit__()
    mine = {"rank": rank, "total_ms": tot / steps, "score_kernel_ms": ker / steps, "merge_ms": mrg / steps,
            "posting_bytes": int(pb)}
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    t = torch.tensor([tot, ker], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot, ker = float(t[0]), float(t[1])
    out = {"value": B * steps / (tot / 1e3), "ms_per_step": tot / steps, "score_kernel_ms": ker / steps,
           "posting_bytes": int(pb), "scorevec_bytes": int(sb), "gpu_launches": int(launches),
           "clocks": clk.summary() if clk else None, "per_rank": per_rank,
           "ids": ids.cpu().numpy() if rank == 0 else None}
    if world > 1:
        out["gather_bytes_per_step"] = int(world * B * k * 8)
        out["rank0_merge_ms"] = per_rank[0]["merge_ms"]
    if e2e:
        h_off = torch.from_numpy(qoff.astype(np.uint64)).pin_memory()
        h_tok = torch.from_numpy(qtok.astype(np.uint32)).pin_memory()
        h_ids = torch.empty((B, k), dtype=torch.uint32).pin_memory()
        h_sc = torch.empty((B, k), dtype=torch.float32).pin_memory()

        def call():
            check(L.sl_retrieve_batch(idx.handle, h_off.data_ptr(), h_tok.data_ptr(), B, k, 1, SL_MEM_HOST,
                                      h_ids.data_ptr(), h_sc.data_ptr()))
        for _ in range(warmup):
            call()
        barrier()
        e2e_s = 0.0
        for _ in range(steps):
            flush.zero_()
            barrier()
            t0 = time.perf_counter()
            call()
            barrier()
            e2e_s += time.perf_counter() - t0
        e = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(e, op=dist.ReduceOp.MAX)
        out["e2e"] = {"value": B * steps / float(e.item()), "unit": "queries/s",
                      "h2d_bytes_per_step": int(h_off.numel() * 8 + h_tok.numel() * 4),
                      "d2h_bytes_per_step": int(B * k * 8)}
    return out


def unique_bytes(idx, qtok, B, V, N_local):
    """8 B x the postings of the batch's distinct tokens + the per-query score vectors."""
    from paper_2407_03618_b200._lib import SL_MEM_HOST, check, lib
    indptr = np.empty(V + 1, np.uint64)
    check(lib().sl_index_export(idx.handle, SL_MEM_HOST, indptr.ctypes.data, None, None, None, None, None, None))
    nnz_t = np.diff(indptr.astype(np.int64))
    return 8 * int(nnz_t[np.unique(qtok)].sum()) + 4 * N_local * B


def extra_block(L, sh, cfg_i, k, variant, args, world, rank, flush, hbm, hbm_src, sms, qrange=None, probe=False):
    """One more workload of the same JSON line: device-timed value (+ e2e), build, per-rank times."""
    from paper_2407_03618_b200 import synth
    qoff, qtok = synth.queries(sh.cfg, sh.cdf, *(qrange or (0, None)))
    B = len(qoff) - 1
    r = time_retrieval(L, sh.idx, qoff, qtok, k, args.steps, args.warmup, rank, world, flush)
    blk = {"config": bench_config(cfg_i, k, variant, sh.cfg.num_docs, sh.cfg.vocab, sh.T_total, B),
           "value": r["value"], "unit": "queries/s", "ms_per_step": r["ms_per_step"],
           "score_kernel_ms": r["score_kernel_ms"], "e2e": r["e2e"], "index_build": sh.build_block(hbm),
           "gpu_launches": r["gpu_launches"]}
    if world > 1:
        blk.update(per_rank=r["per_rank"], gather_bytes_per_step=r["gather_bytes_per_step"],
                   rank0_merge_ms=r["rank0_merge_ms"])
    if probe and rank == 0:
        alg = r["posting_bytes"] + r["scorevec_bytes"]
        blk["roofline"] = physical_roofline(ncu_probe(cfg_i, k, variant, args.dense_density), r["score_kernel_ms"],
                                            alg, unique_bytes(sh.idx, qtok, B, sh.cfg.vocab,
                                                              sh.info.num_docs_local), hbm, hbm_src, sms)
    return blk


def shard_projection_block(L, sh, args, flush):
    """Per-GPU work of an N-way document sharding, measured on this one GPU (N = 2, 4, 8): shard 0
    of the token-balanced split is built with the corpus-wide statistics of the full index (what a
    rank computes after the NCCL all-reduce), the whole query batch is scored on it (device-timed
    like the headline), and the rank-0 merge of N x B x k candidate keys is timed on N copies of
    that shard's keys. Not an N-GPU measurement: the NCCL gather of the keys is not included
    (its bytes are reported)."""
    import torch
    from paper_2407_03618_b200 import BM25Params, Variant, build_index, shard_ranges, synth
    from paper_2407_03618_b200._lib import SL_MEM_DEVICE, SL_MEM_HOST, check
    cfg, k = sh.cfg, args.k
    V, N = cfg.vocab, cfg.num_docs
    df = np.empty(V, np.uint32)
    check(L.sl_index_export(sh.idx.handle, SL_MEM_HOST, None, None, None, df.ctypes.data, None, None, None))
    offsets = synth.doc_offsets(cfg)
    T = int(offsets[-1])
    qoff, qtok = synth.queries(cfg, sh.cdf)
    B = len(qoff) - 1
    d_off = torch.from_numpy(qoff.astype(np.uint64)).cuda()
    d_tok = torch.from_numpy(qtok.astype(np.uint32)).cuda()
    p = BM25Params(Variant[args.variant], 1.5, 0.75, VARIANT_DELTA[args.variant])
    out = {"note": "shard 0 of an N-way token-balanced document sharding on ONE GPU, corpus-wide statistics; "
                   "per_rank = its device-timed retrieve_batch of the whole batch; merge = rank-0 merge of N x B "
                   "x k keys on this GPU; the NCCL gather (gather_bytes) is not measured",
           "config": f"c{args.config} {args.variant} top-{k}, {B} queries"}
    for f in (2, 4, 8):
        d0, d1 = shard_ranges(offsets, f)[0]
        o0, o1 = int(offsets[d0]), int(offsets[d1])
        tok = torch.empty(max(1, o1 - o0), dtype=torch.uint32, device="cuda")
        synth.tokens_device(cfg, sh.cdf, o0, o1 - o0, tok.data_ptr())
        loff = torch.from_numpy((offsets[d0:d1 + 1] - np.uint64(o0)).astype(np.uint64)).cuda()
        with build_index(loff, tok, V, p, doc_base=d0, dense_min_density=args.dense_density,
                         global_stats=(df, N, T)) as ix:
            r = time_retrieval(L, ix, qoff, qtok, k, args.steps, args.warmup, 0, 1, flush, e2e=False)
            keys = torch.empty((B, k), dtype=torch.int64, device="cuda")
            qc = torch.empty(B, dtype=torch.float64, device="cuda")
            check(L.sl_retrieve_local(ix.handle, d_off.data_ptr(), d_tok.data_ptr(), B, k, SL_MEM_DEVICE,
                                      keys.data_ptr(), qc.data_ptr()))
        del tok, loff
        allk = keys.unsqueeze(0).repeat(f, 1, 1).contiguous()
        ids = torch.empty((B, k), dtype=torch.uint32, device="cuda")
        sc = torch.empty((B, k), dtype=torch.float32, device="cuda")
        ms = []
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            check(L.sl_merge_candidates(allk.data_ptr(), f, B, k, qc.data_ptr(), SL_MEM_DEVICE, 0, ids.data_ptr(),
                                        sc.data_ptr()))
            torch.cuda.synchronize()
            if i >= args.warmup:
                ms.append((time.perf_counter() - t0) * 1e3)
        merge_ms = float(np.median(ms))
        out[f"N{f}"] = {"docs": int(d1 - d0), "per_rank_qps": r["value"], "per_rank_ms": r["ms_per_step"],
                        "merge_ms": merge_ms, "gather_bytes": int(f * B * k * 8),
                        "projected_qps_before_gather": B / ((r["ms_per_step"] + merge_ms) / 1e3)}
        del allk, keys, qc
        torch.cuda.empty_cache()
    return out


def run_ncu_child(args):
    """--ncu-child: build the workload's index and run ONE retrieve_batch (profiled by ncu_probe)."""
    import torch
    from paper_2407_03618_b200 import synth
    from paper_2407_03618_b200._lib import lib
    torch.cuda.set_device(0)
    sh = Shard(args.config, args.variant, 1, 0, 0, None, args.dense_density)
    qoff, qtok = synth.queries(sh.cfg, sh.cdf)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    time_retrieval(lib(), sh.idx, qoff, qtok, args.k, 1, 0, 0, 1, flush, e2e=False)
    sh.close()
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2407_03618_b200 import Comm, synth
    from paper_2407_03618_b200._lib import lib

    world, rank, local = dist_setup()
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    if world > 1:  # communicator INIT lines (nranks) in the log: the driver's evidence of a real multi-rank run
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = lib()
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    hbm, hbm_src = peaks()
    comm = None
    if world > 1:
        uid = [Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = Comm(uid[0], world, rank, local)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    # ---- headline workload
    sh = Shard(args.config, args.variant, world, rank, local, comm, args.dense_density, args.shard_of,
               args.shard_index)
    qoff, qtok = synth.queries(sh.cfg, sh.cdf)
    B, k = len(qoff) - 1, args.k
    r = time_retrieval(L, sh.idx, qoff, qtok, k, args.steps, args.warmup, rank, world, flush, clock_dev=local)
    line = None
    if rank == 0:
        alg = r["posting_bytes"] + r["scorevec_bytes"]
        cfgd = bench_config(args.config, k, args.variant, sh.cfg.num_docs, sh.cfg.vocab, sh.T_total, B)
        if args.shard_of > 1:
            cfgd["simulated_shard"] = (f"{args.shard_index} of {args.shard_of} (docs {sh.d0}..{sh.d1}; shard-local "
                                       "df/N statistics; value is per-GPU)")
        line = {
            "metric": METRIC, "value": r["value"], "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 accumulate (f64 build math)",
            "data": "synthetic (seeded Zipf corpus/queries, BASELINE.md §5; BEIR absent)",
            "config": cfgd, "parallelism": f"document-sharded over {world} GPU(s) (one process per GPU)",
            "timing": "CUDA events on the library stream, L2 flushed between steps (256 MiB memset), max over ranks",
            "index_tokens_per_s": sh.T_total / (sh.build_ms / 1e3),
            "index_build": sh.build_block(hbm),
            "score_kernel_ms_per_step": r["score_kernel_ms"],
            "e2e": r["e2e"], "gpu_launches": r["gpu_launches"], "clocks": r["clocks"],
        }
        if world > 1:
            line.update(per_rank=r["per_rank"], gather_bytes_per_step=r["gather_bytes_per_step"],
                        rank0_merge_ms=r["rank0_merge_ms"])
        if world == 1 and not args.no_ncu:
            line["roofline"] = physical_roofline(ncu_probe(args.config, k, args.variant, args.dense_density),
                                                 r["score_kernel_ms"], alg,
                                                 unique_bytes(sh.idx, qtok, B, sh.cfg.vocab, sh.info.num_docs_local),
                                                 hbm, hbm_src, sms)
    head_ids = r["ids"]
    blocks = {}
    if not args.no_extra and args.shard_of == 1:
        if args.config == 2 and args.variant == "lucene":
            blocks["c2_top100"] = extra_block(L, sh, 2, 100, "lucene", args, world, rank, flush, hbm, hbm_src, sms)
        if world == 1 and not args.no_projection:
            blocks["shard_projection"] = shard_projection_block(L, sh, args, flush)
        sh.close()
        if args.config == 2 and world == 1:  # c3: the variant sweep on c2's corpus
            for v in ("robertson", "atire", "bm25l", "bm25plus"):
                s3 = Shard(2, v, world, rank, local, comm, args.dense_density)
                blocks[f"c3_{v}_top10"] = extra_block(L, s3, 3, 10, v, args, world, rank, flush, hbm, hbm_src, sms)
                s3.close()
        if args.config != 4:  # c4 (configs[3]) at every N: the largest corpus the 1/2/4/8 curve covers
            s4 = Shard(4, "lucene", world, rank, local, comm, args.dense_density)
            blocks["c4_top1000"] = extra_block(L, s4, 4, 1000, "lucene", args, world, rank, flush, hbm, hbm_src, sms,
                                               qrange=(0, 8192), probe=(world == 1 and not args.no_ncu))
            s4.close()
        if world == 8 or args.c5:  # c5 (configs[4]) is an 8-GPU config
            s5 = Shard(5, "lucene", world, rank, local, comm, args.dense_density)
            blocks["c5_top100"] = extra_block(L, s5, 5, 100, "lucene", args, world, rank, flush, hbm, hbm_src, sms)
            s5.close()
    else:
        sh.close()
    if rank == 0:
        line.update(blocks)
        if world == 1 and not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            corp = cpu_corpus(args.config)
            ox, build_s = cpu_index(corp, args.variant)
            nq = min(B, args.cpu_sample)
            qps1, ids1 = cpu_qps(ox, qoff, qtok, nq, k, 1)
            nq_all = min(B, 16 * args.cpu_sample)
            qpsn, _ = cpu_qps(ox, qoff, qtok, nq_all, k, cores)
            line["cpu_baseline"] = {"value": qpsn, "unit": "queries/s", "cores": cores, "kind": "port",
                                    "sample": f"first {nq_all} queries of c{args.config}, workers={cores}, full "
                                              f"index; CPU build (1 thread) {build_s:.1f}s = "
                                              f"{int(corp.offsets[-1]) / build_s:.3g} tokens/s",
                                    "single_thread": {"value": qps1, "unit": "queries/s", "cores": 1,
                                                      "sample": f"first {nq} queries, workers=1 (the paper's "
                                                                "single-threaded QPS)"},
                                    "host": host_info()}
            agree = float(np.mean(head_ids[:nq] == ids1))
            line["parity_sample"] = {"queries": nq, "top_k_id_agreement": agree}
        if world == 1 and not args.no_text:
            line["text_pipeline"] = text_pipeline_block(args.config, hbm)
        print(json.dumps(line), flush=True)
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
    ap.add_argument("--no-extra", action="store_true", help="skip the c2 top-100 / c3 / c4 / c5 blocks")
    ap.add_argument("--no-ncu", action="store_true", help="skip the in-run ncu counters (roofline traffic)")
    ap.add_argument("--c5", action="store_true", help="add the c5 block below 8 GPUs (each rank holds 1/N)")
    ap.add_argument("--no-projection", action="store_true",
                    help="skip the one-GPU per-rank measurement of the 2/4/8-way document sharding")
    ap.add_argument("--cpu-sample", type=int, default=64)
    ap.add_argument("--ref-sample", type=int, default=0, help="reference arm: queries per step (0 = the whole batch)")
    ap.add_argument("--shard-of", type=int, default=1, help="build one shard of an N-way doc sharding (1 GPU)")
    ap.add_argument("--shard-index", type=int, default=0)
    ap.add_argument("--ncu-child", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.ncu_child:
        return run_ncu_child(args)
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    return run_reference(args) if args.impl == "reference" else run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
