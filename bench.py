#!/usr/bin/env python
"""bench.py -- FlatQuant online hot path on B200: prefill tokens/s of all layer linears.

One step = the whole hot path over one batch of synthetic tokens:
for every linear of the configuration, fq_transform_quant (Kronecker transform + clip + INT4
quantize/pack) followed by fq_w4a4_linear (tcgen05 W4A4 GEMM + dequant epilogue) -- or, at decode
sizes (T <= 64, 64 x 64 or 112 x 128 decomposition), fq_flatquant_linear, which runs both in ONE fused launch
(NEXT-4(i); --no-fused keeps the two calls).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

N > 1 runs one process per GPU under torchrun (NCCL).  Launched without torchrun, `--gpus N`
re-executes itself under `python -m torch.distributed.run --nproc-per-node N`; launched by
torchrun, WORLD_SIZE must equal N (anything else is an error, never a silent 1-GPU run).
Sharding: tokens are independent, so every rank owns a contiguous block of
the global batch (paper_2410_09426_b200.sharding.shard_range), weights and transforms are
replicated, and the timed path has no collective.  C1-C4 scale weakly (every rank processes the
configuration's T tokens, rows [r T, (r+1) T) of an N T-token batch); C5, whose BASELINE config
is a 16 x 2048-token batch sharded across the GPUs, scales strongly (T / N tokens per rank).
The step time is the max over ranks.  After the timed region (untimed), an NCCL all-gather of
the first linear's output is checked bit for bit against rank 0's own recompute of the last
rank's shard.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
INT8_PER_BF16 = 2.0          # nominal dense ratio (4.5 / 2.25 POPS), B200_PROFILING.md


def ncu_traffic(cfg_name, linears, kind):
    """DRAM bytes (read + write) of one step's `kind` launches ("gemm" or "tq") from the committed
    ncu --set full captures (profiles/ncu_traffic.json, scripts/make_profiles.py), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    # the captures are of C3's shapes (gemm_*, tq_*) and of C4's fused decode linears (fused_*);
    # C2's one linear (2048 x 4096 -> 4096, 64 x 64) is C3's o_proj shape, so its capture serves
    if (cfg_name, kind) not in (("C2", "gemm"), ("C2", "tq"), ("C3", "gemm"), ("C3", "tq"), ("C4", "fused")) \
            or not os.path.exists(path):
        return None
    t = json.load(open(path))
    keys = [f"{kind}_P_o" if cfg_name == "C2" else f"{kind}_{lin.name}" for lin in linears]
    if not all(k in t for k in keys):
        return None
    return {"bytes_per_step": int(sum(t[k]["dram_bytes"] for k in keys)),
            "source": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum, one launch per linear: "
                      + ", ".join(sorted({t[k]["capture"].split(":")[0] for k in keys}))}


def peaks():
    if os.path.exists(PEAKS_PATH):
        p = json.load(open(PEAKS_PATH))
        return p, "measured (MEASURED_PEAKS.json)"
    return dict(FALLBACK), "fallback (B200_PROFILING.md)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--alpha", type=float, default=0.9)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-streams", type=int, default=4, help="streams the e2e step's linears rotate over")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp16", action="store_true")
    ap.add_argument("--no-kv", action="store_true", help="skip the KV-cache quantization measurement")
    ap.add_argument("--no-verify", action="store_true", help="N > 1: skip the untimed all-gather check")
    ap.add_argument("--no-fig6", action="store_true", help="skip the per-transform in-step overhead steps")
    ap.add_argument("--no-fused", action="store_true",
                    help="decode: call fq_transform_quant + fq_w4a4_linear instead of the fused fq_flatquant_linear")
    return ap.parse_args()


def launch_or_check_world(args):
    """--gpus N: re-exec under torchrun if not already a torchrun rank; else WORLD_SIZE must be N."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is None:
        if args.gpus > 1 and args.impl == "ours":
            import socket
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
            sys.stderr.write("[bench] --gpus %d without torchrun: launching %s\n" % (args.gpus, " ".join(cmd)))
            sys.stderr.flush()
            os.execv(sys.executable, cmd)
        return
    if int(ws) != args.gpus:
        sys.stderr.write(f"[bench] error: --gpus {args.gpus} but WORLD_SIZE={ws}: refusing to report a "
                         f"{ws}-process run as {args.gpus} GPUs\n")
        sys.exit(2)


# ------------------------------------------------------------------------ clocks sampler
class Clocks:
    """nvidia-smi sampler (100 ms) started before the warm-up; the summary keeps the samples
    taken inside the timed window (padded by 0.3 s, since one window can be shorter than a
    sampling period)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append((time.time(), parts))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        time.sleep(0.35)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for t, r in self.rows if self.t0 is not None and self.t0 - 0.3 <= t <= self.t1 + 0.3]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        sm = [v for v in (num(r[0]) for r in rows) if v is not None]
        mx = [v for v in (num(r[1]) for r in rows) if v is not None]
        pw = [v for v in (num(r[6]) for r in rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------------------ workload
STRONG = {"C5"}        # configs whose global batch is split across the ranks (BASELINE config 5)


def token_block(cfg_name, rank, world):
    """(lo, hi, global_T): the rows of the global batch that `rank` owns."""
    from paper_2410_09426_b200.sharding import shard_range
    T = synth.config(cfg_name)["T"]
    total = T if cfg_name in STRONG else T * world
    lo, hi = shard_range(total, rank, world)
    return lo, hi, total


def build_workload(cfg_name, rank, world, dev, torch, fq):
    cfg = synth.config(cfg_name)
    lo, hi, _ = token_block(cfg_name, rank, world)
    T = hi - lo
    layers = []
    for lin in cfg["linears"]:
        n1, n2, N, K = lin.n1, lin.n2, lin.N, lin.K
        x = torch.from_numpy(synth.activations(hi, K, seed=1000, tag=lin.name, rows=range(lo, hi))).to(dev)
        p1 = torch.from_numpy(synth.well_conditioned(n1, seed=0, tag=lin.name + "/p1")).to(dev)
        p2 = torch.from_numpy(synth.well_conditioned(n2, seed=0, tag=lin.name + "/p2")).to(dev)
        w = torch.from_numpy(synth.weights(N, K, seed=0, tag=lin.name)).to(dev)
        qw, sw = fq.prepare_weight(w, n1, n2, p1, p2, 1.0)          # offline weight side on the GPU
        layers.append(dict(lin=lin, x=x, p1=p1, p2=p2, w=w, qw=qw, sw=sw,
                           q=torch.empty((T, K // 2), dtype=torch.uint8, device=dev),
                           s=torch.empty((T,), dtype=torch.float32, device=dev),
                           y=torch.empty((T, N), dtype=torch.float16, device=dev)))
    return cfg, layers, T


def fused_linear(T, lin):
    """The library runs fq_flatquant_linear as ONE fused launch (transform + quantize inside the
    decode GEMM, NEXT-4(i)) for T <= 64 with the 64 x 64 decomposition and fp16 activations
    (fq_gemm_dec.cu FUSED); the bench checks this against its launch count."""
    return T <= 64 and (lin.n1, lin.n2) in ((64, 64), (64, 128), (112, 128))


def fused_bytes(T, lin):
    """Algorithmic bytes of one fused decode linear: the transform's (X in, codes + scales out to
    the caller's workspace, P1, P2) plus the GEMM's weights, weight scales and output; the codes are
    read back from L2 inside the launch, so they count once."""
    return tq_bytes(T, lin) + gemm_min_bytes(T, lin) - (T * lin.K // 2 + 4 * T)


def tq_bytes(T, lin):
    return T * (2 * lin.K + lin.K // 2 + 4) + 2 * (lin.n1 ** 2 + lin.n2 ** 2)


def tq_flops(T, lin):
    return 2 * T * lin.K * (lin.n1 + lin.n2)


def gemm_ops(T, lin):
    return 2 * T * lin.N * lin.K


def gemm_min_bytes(T, lin):
    """Compulsory HBM bytes of one W4A4 GEMM: packed codes of A and W, scales, fp16 output."""
    return T * lin.K // 2 + lin.N * lin.K // 2 + 4 * (T + lin.N) + 2 * T * lin.N


# ------------------------------------------------------------------------ oracle (CPU) timing
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count()


def cpu_oracle_rate(cfg_name, sample_tokens, alpha, budget_s=12.0, threads=None):
    """The float64 oracle as it stands, on a bounded token sample of the same workload; with
    `threads`, its BLAS pool is limited to that many threads (threadpoolctl)."""
    import contextlib

    import oracle as O
    ctx = contextlib.nullcontext()
    if threads is not None:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(limits=threads)
    cfg = synth.config(cfg_name)
    prepared = []
    for lin in cfg["linears"]:
        x = synth.activations(sample_tokens, lin.K, seed=1000, tag=lin.name)
        p1 = synth.well_conditioned(lin.n1, seed=0, tag=lin.name + "/p1")
        p2 = synth.well_conditioned(lin.n2, seed=0, tag=lin.name + "/p2")
        w = synth.weights(lin.N, lin.K, seed=0, tag=lin.name)
        qw, sw, _ = O.prepare_weight(w, p1, p2, 1.0)                 # offline, untimed
        prepared.append((x, p1, p2, qw, sw))
    with ctx:
        cores = threads if threads is not None else blas_threads()
        done, t0 = 0, time.perf_counter()
        while True:
            for x, p1, p2, qw, sw in prepared:
                qa, sa, _ = O.transform_quant(x, p1, p2, alpha)
                O.dequant(O.int_gemm(qa, qw), sa, sw)
            done += sample_tokens
            el = time.perf_counter() - t0
            if el >= budget_s or done >= 4 * sample_tokens:
                break
    return done / el, cores, f"{sample_tokens} tokens x {done // sample_tokens} passes of all {cfg_name} linears " \
                             f"(transform+quant, int GEMM, dequant; weight prep untimed), {el:.1f} s"


def cpu_baseline(cfg_name, alpha):
    """all-core and 1-thread rates of the oracle, with the host's core count and CPU model"""
    rate, cores, sample = cpu_oracle_rate(cfg_name, 128, alpha)
    r1, _, s1 = cpu_oracle_rate(cfg_name, 32, alpha, threads=1)
    return {"value": round(rate, 2), "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": sample,
            "nproc": os.cpu_count(), "cpu_model": cpu_model(),
            "one_thread": {"value": round(r1, 2), "unit": "tokens/s", "cores": 1, "sample": s1}}


# ------------------------------------------------------------------------ our implementation
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2410_09426_b200 as fq

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    fq.load()
    if os.environ.get("FQ_GEMM_IMPL"):                     # testing aid: 0 pair (default), 1 mma.sync, 2 1-CTA
        fq.fq_set_gemm_impl(int(os.environ["FQ_GEMM_IMPL"]))
    if os.environ.get("FQ_TQ_IMPL"):                       # testing aid: 0 default, 1 mma.sync, 2 CUDA cores
        fq.fq_set_tq_impl(int(os.environ["FQ_TQ_IMPL"]))

    cfg, layers, T = build_workload(args.config, rank, world, dev, torch, fq)
    lo, hi, total_T = token_block(args.config, rank, world)
    scaling = "strong" if args.config in STRONG else "weak"
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # 2x L2 (126 MB)
    flush_sum = torch.empty((), dtype=torch.float32, device=dev)

    def flush_l2():
        # write then read 256 MiB: the dirty lines of the write are evicted by the read, so the
        # next kernel finds the L2 full of clean lines it does not need (no write-back charged to it)
        flush.zero_()
        torch.sum(flush, dim=0, out=flush_sum)
        torch.cuda._sleep(400_000)    # lets the host enqueue the whole step before the GPU reaches it

    fused = [not args.no_fused and fused_linear(T, L["lin"]) for L in layers]

    def step(evs=None, tq_mask=None, gemm=True, po_paper=None):
        for i, L in enumerate(layers):
            lin = L["lin"]
            if fused[i] and gemm and (tq_mask is None or tq_mask[i]) and po_paper is None:
                # the whole linear in one launch (events around it in the GEMM slot)
                if evs is not None:
                    evs[2 * i + 1][0].record(stream)
                fq.fq_flatquant_linear(L["x"], lin.n1, lin.n2, L["p1"], L["p2"], args.alpha, L["qw"], L["sw"],
                                       L["y"], L["q"], L["s"])
                if evs is not None:
                    evs[2 * i + 1][1].record(stream)
                continue
            if tq_mask is None or tq_mask[i]:
                if evs is not None:
                    evs[2 * i][0].record(stream)
                if po_paper is not None and lin.name == "P_o":
                    fq.fq_transform_quant(L["x"], 32, 128, po_paper, None, args.alpha, L["q"], L["s"])
                else:
                    fq.fq_transform_quant(L["x"], lin.n1, lin.n2, L["p1"], L["p2"], args.alpha, L["q"], L["s"])
                if evs is not None:
                    evs[2 * i][1].record(stream)
            if gemm:
                if evs is not None:
                    evs[2 * i + 1][0].record(stream)
                fq.fq_w4a4_linear(L["q"], L["s"], L["qw"], L["sw"], L["y"])
                if evs is not None:
                    evs[2 * i + 1][1].record(stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    from paper_2410_09426_b200 import sharding

    def max_over_ranks(v):
        return sharding.max_over_ranks(v, dev)

    def timed_steps(n, **kw):
        """n steps, L2 flushed before each (flush untimed); returns the summed step time (ms).
        One untimed step first: a variant's first launches pay one-time host costs (kernel
        attributes, occupancy queries) that the device sleep after the flush does not cover."""
        step(**kw)
        tot = 0.0
        for _ in range(n):
            flush_l2()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step(**kw)
            b.record(stream)
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
        return tot

    clk = Clocks(local).start()
    t_w = time.time()
    w = 0
    while w < max(args.warmup, 3) or time.time() - t_w < 1.0:      # >= 1 s soak so clocks settle
        flush_l2()
        step()
        w += 1
        if w % 50 == 0:
            torch.cuda.synchronize()
    barrier()

    # ---- timed region: K steps between barriers.  Pass 1 times the step alone (first kernel start
    #      -> last kernel end, kernels back to back so programmatic dependent launch overlaps their
    #      launches); pass 2 re-runs the K steps with events around every kernel for the per-kernel
    #      roofline numbers (events between kernels serialise them and add ~5 us each, see
    #      `event_overhead`).
    per_kernel = [[0.0, 0.0] for _ in range(2 * len(layers))]
    launches0 = fq.fq_launch_count()
    clk.mark_start()
    t_start = time.time()
    total_ms = timed_steps(args.steps)
    barrier()
    wall_s = time.time() - t_start
    # timed_steps runs one untimed step before the timed ones; every step launches the same kernels
    launches = (fq.fq_launch_count() - launches0) * args.steps // (args.steps + 1)
    for _ in range(args.steps):
        flush_l2()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(2 * len(layers))]
        step(evs)
        torch.cuda.synchronize()
        for k, (ea, eb) in enumerate(evs):
            if k % 2 == 0 and fused[k // 2]:
                continue                                 # fused linear: one launch, in the GEMM slot
            per_kernel[k][0] += ea.elapsed_time(eb)
            per_kernel[k][1] += 1
    barrier()
    clk.mark_end()
    clk.stop()
    my_ms = total_ms / args.steps
    total_ms = max_over_ranks(total_ms)
    ms_per_step = total_ms / args.steps
    value = total_T / (ms_per_step * 1e-3)          # all tokens of all ranks / max-over-ranks step time
    rank_lines = None
    if world > 1:
        props = torch.cuda.get_device_properties(dev)
        bus = float(getattr(props, "pci_bus_id", -1)) * 1000.0 + float(getattr(props, "pci_device_id", 0))
        rows = sharding.rank_table([rank, T, my_ms, props.multi_processor_count, bus], dev)
        rank_lines = [{"rank": int(r[0]), "tokens": int(r[1]), "ms_per_step": round(float(r[2]), 4),
                       "tokens_per_s": round(float(r[1]) / (float(r[2]) * 1e-3), 1), "sms": int(r[3]),
                       "pci": int(r[4])} for r in rows]
    sys.stderr.write(f"[bench] rank {rank}/{world} cuda:{local} {torch.cuda.get_device_name(dev)} "
                     f"backend={'nccl' if world > 1 else 'none'} tokens [{lo},{hi}) of {total_T}: "
                     f"{my_ms:.4f} ms/step\n")

    # ---- kernel-level rooflines ----
    pk, peak_src = peaks()
    gemm_ms = sum(per_kernel[2 * i + 1][0] for i in range(len(layers))) / args.steps
    tq_ms = sum(per_kernel[2 * i][0] for i in range(len(layers))) / args.steps
    g_ops = sum(gemm_ops(T, L["lin"]) for L in layers)
    t_bytes = sum(tq_bytes(T, L["lin"]) for i, L in enumerate(layers) if not fused[i])
    t_flops = sum(tq_flops(T, L["lin"]) for i, L in enumerate(layers) if not fused[i])
    int8_peak, int8_src, int8_alt = int8_peak_tops(pk, peak_src)
    gemm_tops = g_ops / (gemm_ms * 1e-3) / 1e12
    tq_gbs = t_bytes / (tq_ms * 1e-3) / 1e9 if tq_ms > 0 else 0.0
    kernels = {}
    for i, L in enumerate(layers):
        lin = L["lin"]
        tq_i = per_kernel[2 * i][0] / args.steps
        gm_i = per_kernel[2 * i + 1][0] / args.steps
        if fused[i]:
            kernels[lin.name] = {
                "n1xn2": f"{lin.n1}x{lin.n2}", "N": lin.N, "fused": True,
                "linear_us": round(gm_i * 1e3, 2), "linear_gbs": round(fused_bytes(T, lin) / (gm_i * 1e-3) / 1e9, 1),
                "gemm_tops": round(gemm_ops(T, lin) / (gm_i * 1e-3) / 1e12, 1),
                "note": "fq_flatquant_linear: transform + quantize + GEMM + dequant in one launch"}
            continue
        kernels[lin.name] = {
            "n1xn2": f"{lin.n1}x{lin.n2}", "N": lin.N,
            "tq_us": round(tq_i * 1e3, 2), "tq_gbs": round(tq_bytes(T, lin) / (tq_i * 1e-3) / 1e9, 1),
            "tq_tflops": round(tq_flops(T, lin) / (tq_i * 1e-3) / 1e12, 1),
            "gemm_us": round(gm_i * 1e3, 2), "gemm_tops": round(gemm_ops(T, lin) / (gm_i * 1e-3) / 1e12, 1),
            "gemm_gbs": round(gemm_min_bytes(T, lin) / (gm_i * 1e-3) / 1e9, 1),
        }

    # ---- event overhead and a same-byte copy (what an event-timed launch of this size can show) ----
    one = torch.zeros(1, device=dev)
    ev_empty = timed_ms(torch, stream, flush_l2, lambda: one.add_(1), max(5, args.steps))
    cp_bytes = tq_bytes(T, layers[0]["lin"])
    cp_src = torch.empty(cp_bytes // 4, dtype=torch.float16, device=dev)
    cp_dst = torch.empty_like(cp_src)
    ev_copy = timed_ms(torch, stream, flush_l2, lambda: cp_dst.copy_(cp_src), max(5, args.steps))
    del cp_src, cp_dst

    # ---- Fig. 6 analogue and the transforms' in-step cost: the same step
    #      without any transform kernel (GEMMs on the codes already in place: "plain INT4"), and
    #      with exactly one transform kernel added back; the difference is that transform's
    #      marginal cost inside the step (PDL overlap included).  Also the step with the paper's
    #      own o_proj transform P_o (32 x 32) x I_128 in place of the generic 64 x 64.
    fig6 = None
    if not args.no_fig6:
        nl = len(layers)
        reps = max(5, args.steps)
        t_gemm_only = timed_steps(reps, tq_mask=[False] * nl) / reps
        t_full = timed_steps(reps) / reps
        per = {}
        marg_sum = 0.0
        for i, L in enumerate(layers):
            mask = [j == i for j in range(nl)]
            t_i = timed_steps(reps, tq_mask=mask) / reps
            m_i = t_i - t_gemm_only
            marg_sum += m_i
            per[L["lin"].name] = {"transform": f"{L['lin'].n1}x{L['lin'].n2}", "step_ms": round(t_i, 4),
                                  "marginal_us": round(m_i * 1e3, 2),
                                  "slowdown_vs_int4": round(m_i / t_gemm_only, 4),
                                  "marginal_gbs": round(tq_bytes(T, L["lin"]) / max(m_i * 1e-3, 1e-12) / 1e9, 1)}
        fig6 = {"int4_gemm_only_step_ms": round(t_gemm_only, 4), "full_step_ms": round(t_full, 4),
                "total_slowdown_vs_int4": round((t_full - t_gemm_only) / t_gemm_only, 4), "per_transform": per,
                "paper_rtx3090": {"total": 0.07, "P_d": 0.04, "P_o": 0.01,
                                  "source": "PAPER.md:510 (Fig. 6), 529-531; context only"},
                "note": "INT4 = the same W4A4 GEMMs on codes already in HBM (no transform/quantize kernel); "
                        "marginal = step with that one transform+quantize kernel minus the INT4 step"}
        L_o = next((L for L in layers if L["lin"].name == "P_o"), None)
        if L_o is not None and L_o["lin"].K == 4096:
            p_o = torch.linalg.qr(torch.randn((32, 32), generator=torch.Generator(device=dev).manual_seed(7),
                                              device=dev))[0].half().contiguous()
            mask = [L["lin"].name == "P_o" for L in layers]
            t_po = timed_steps(reps, tq_mask=mask, po_paper=p_o) / reps
            fig6["per_transform"]["P_o_paper"] = {
                "transform": "P_o (32x32) x I_128 (p2 = NULL), the paper's online o_proj form (PAPER.md:297, 726)",
                "step_ms": round(t_po, 4), "marginal_us": round((t_po - t_gemm_only) * 1e3, 2),
                "slowdown_vs_int4": round((t_po - t_gemm_only) / t_gemm_only, 4)}
        fig6["in_step_tq_gbs"] = round(t_bytes / max(marg_sum * 1e-3, 1e-12) / 1e9, 1)

    # ---- FP16 baseline (torch.matmul / cuBLAS on the same shapes), context for "vs FP16" ----
    fp16 = None
    if not args.no_fp16:
        xs = [L["x"] for L in layers]
        ws = [L["w"] for L in layers]
        f_ms = timed_ms(torch, stream, flush_l2, lambda: [torch.matmul(x, w.t()) for x, w in zip(xs, ws)],
                        max(5, args.steps // 2))
        fp16_ms = max_over_ranks(f_ms)
        fp16 = {"ms_per_step": round(fp16_ms, 4), "tokens_per_s": round(total_T / (fp16_ms * 1e-3), 1),
                "speedup_ours_vs_fp16": round(fp16_ms / ms_per_step, 3)}

    # ---- KV-cache quantization, measured beside the step (not part of it).
    #      Keys (P_h) and values (P = I) of LLaMA-3-8B (8 KV heads x head_dim 128) for two sizes:
    #      this step's tokens, and the paper's decoding setting, batch 64 x 2048 tokens.
    kv = None
    if not args.no_kv:
        H, D = 8, 128
        gk = torch.Generator(device=dev).manual_seed(1234 + rank)
        ph = torch.linalg.qr(torch.randn((D, D), generator=gk, device=dev))[0].half().contiguous()
        eye = torch.eye(D, device=dev).half()
        kv = {"kernel": "fq_kv_quant (tcgen05 kind::f16, K with P_h + V with P = I)", "head_dim": D, "bound": "hbm",
              "peak": pk["hbm_gbs"], "unit": "GB/s", "l2": "flushed (write + read) before every timed K+V pair",
              "sizes": []}
        for label, R in ((f"step: {T} tokens x {H} heads", T * H), (f"batch 64 x 2048 tokens x {H} heads", 64 * 2048 * H)):
            kk = torch.randn((R, D), generator=gk, device=dev).half()
            vv = torch.randn((R, D), generator=gk, device=dev).half()
            outs = [(torch.empty((R, D // 2), dtype=torch.uint8, device=dev), torch.empty(R, device=dev),
                     torch.empty(R, dtype=torch.int8, device=dev)) for _ in range(2)]

            def kv_step():
                fq.fq_kv_quant(kk, ph, 0.95, *outs[0])
                fq.fq_kv_quant(vv, eye, 0.95, *outs[1])

            kv_ms = timed_ms(torch, stream, flush_l2, kv_step, max(5, args.steps))
            kv_bytes = 2 * R * (2 * D + D // 2 + 4 + 1)
            kv_gbs = kv_bytes / (kv_ms * 1e-3) / 1e9
            kv["sizes"].append({"workload": label, "head_vectors": 2 * R, "us": round(kv_ms * 1e3, 2),
                                "achieved": round(kv_gbs, 1), "frac": round(kv_gbs / pk["hbm_gbs"], 4),
                                "algorithmic_bytes": int(kv_bytes)})
            del kk, vv, outs

    # ---- e2e: through the public C ABI with HOST buffers (H2D + hot path + D2H per step) ----
    e2e = None
    if not args.no_e2e:
        hx = [L["x"].cpu().pin_memory() for L in layers]
        hy = [torch.empty(L["y"].shape, dtype=L["y"].dtype).pin_memory() for L in layers]
        dx = [torch.empty_like(L["x"]) for L in layers]

        # one stream per linear (the four linears of a step are independent inputs here): every
        # H2D copy is queued at once and each linear's D2H overlaps the others' copies and compute
        # (PCIe is full duplex); every linear has its own staging buffers.  The step ends when all
        # streams are done.  Measured e2e (same box): C4 1 / 2 / 4 streams 0.190 / 0.215 / 0.240 M
        # tokens/s, C3 0.369 / 0.520 / 0.540 M.  (Splitting each linear into 4 token chunks was
        # measured slower: 0.47 vs 0.51 M tokens/s on C3.)
        e2e_streams = [torch.cuda.Stream(device=dev) for _ in range(max(1, args.e2e_streams))]

        def e2e_step():
            start = torch.cuda.Event()
            start.record(stream)
            for st in e2e_streams:
                st.wait_event(start)
            for i, (L, x_h, y_h, x_d) in enumerate(zip(layers, hx, hy, dx)):
                lin = L["lin"]
                fq.fq_flatquant_linear_host(x_h, x_d, lin.n1, lin.n2, L["p1"], L["p2"], args.alpha, L["qw"], L["sw"],
                                            y_h, L["y"], L["q"], L["s"], stream=e2e_streams[i % len(e2e_streams)], sync=False)
            for st in e2e_streams:
                done = torch.cuda.Event()
                done.record(st)
                stream.wait_event(done)

        for _ in range(2):
            e2e_step()
        barrier()
        e_ms = []
        for _ in range(max(3, args.steps // 2)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e2e_step()
            b.record(stream)
            torch.cuda.synchronize()
            e_ms.append(a.elapsed_time(b))
        e2e_step_ms = max_over_ranks(sum(e_ms)) / len(e_ms)
        e2e = {"value": round(total_T / (e2e_step_ms * 1e-3), 1), "unit": "tokens/s",
               "ms_per_step": round(e2e_step_ms, 4),
               "h2d_bytes_per_step": int(sum(x.numel() * x.element_size() for x in hx)),
               "d2h_bytes_per_step": int(sum(y.numel() * y.element_size() for y in hy))}

    # ---- verification (untimed, N > 1): all-gather the first linear's output over NCCL; rank 0
    #      recomputes the LAST rank's shard itself (same inputs regenerated from the seeded
    #      streams, same kernels) and compares bit for bit; every rank checks its own block.
    verify = None
    if world > 1 and not args.no_verify:
        L0 = layers[0]
        lin = L0["lin"]
        step()
        torch.cuda.synchronize()

        def recompute_last(rlo, rhi):
            xr = torch.from_numpy(synth.activations(rhi, lin.K, seed=1000, tag=lin.name, rows=range(rlo, rhi))).to(dev)
            yr = fq.flatquant_linear(xr, lin.n1, lin.n2, L0["p1"], L0["p2"], args.alpha, L0["qw"], L0["sw"])
            torch.cuda.synchronize()
            return yr

        verify = sharding.verify_gather(L0["y"], total_T, recompute_last)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, args.alpha)

    gemm_traffic = ncu_traffic(args.config, [L["lin"] for L in layers], "fused" if all(fused) else "gemm")
    tq_traffic = ncu_traffic(args.config, [L["lin"] for L in layers], "tq")
    decode = T <= 64     # decode step (C4): the GEMM streams the weights, HBM-bound (SURVEY 8(a) sizes)
    g_bytes = sum(fused_bytes(T, L["lin"]) if fused[i] else gemm_min_bytes(T, L["lin"]) for i, L in enumerate(layers))
    if decode:
        g_gbs = g_bytes / (gemm_ms * 1e-3) / 1e9
        kname = "fq_w4a4_linear (decode kernel: tcgen05 kind::i8, cluster split-K)"
        if any(fused):
            kname = ("decode GEMM launches: fq_flatquant_linear fused (transform + tcgen05 kind::i8 GEMM, "
                     + ", ".join(L["lin"].name for i, L in enumerate(layers) if fused[i]) + ")")
            if not all(fused):
                kname += (", fq_w4a4_linear ("
                          + ", ".join(L["lin"].name for i, L in enumerate(layers) if not fused[i]) + ")")
        roof = {"bound": "hbm", "kernel": kname,
                "achieved": round(g_gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(g_gbs / pk["hbm_gbs"], 4), "traffic": gemm_traffic,
                "per": "aggregate of the step's GEMM launches (sum of compulsory bytes / sum of their durations; "
                       "a fused launch counts its transform's bytes too)",
                "algorithmic_bytes_per_step": int(g_bytes), "tops": round(gemm_tops, 1),
                "peak_source": f"{peak_src}: hbm_gbs"}
    else:
        roof = {"bound": "tensor", "kernel": "fq_w4a4_linear (tcgen05 kind::i8)",
                "achieved": round(gemm_tops, 1), "peak": round(int8_peak, 1), "unit": "TOPS",
                "frac": round(gemm_tops / int8_peak, 4), "traffic": gemm_traffic,
                "per": "aggregate of the step's GEMM launches (sum of 2TNK / sum of their durations)",
                "algorithmic_bytes_per_step": int(g_bytes), "peak_source": int8_src}
        if int8_alt:
            roof["alt_peaks"] = dict(int8_alt)
            for k in ("tcgen05_issue_loop_tops", "cublaslt_int8_8192_tops"):
                if int8_alt.get(k):
                    roof["alt_peaks"]["frac_vs_" + k.replace("_tops", "")] = round(gemm_tops / int8_alt[k], 4)
    tq_roof = {"bound": "hbm", "kernel": "fq_transform_quant", "achieved": round(tq_gbs, 1),
               "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(tq_gbs / pk["hbm_gbs"], 4),
               "traffic": tq_traffic, "algorithmic_bytes_per_step": int(t_bytes),
               "tflops": round(t_flops / (tq_ms * 1e-3) / 1e12, 1) if tq_ms > 0 else None,
               "per": "sum of algorithmic bytes / sum of event-timed launch durations (pass 2)",
               "event_overhead": {"empty_kernel_us": round(ev_empty * 1e3, 2),
                                  "same_bytes_copy_us": round(ev_copy * 1e3, 2),
                                  "same_bytes_copy_gbs": round(cp_bytes / (ev_copy * 1e-3) / 1e9, 1),
                                  "note": "an event-bracketed empty kernel and a torch copy moving one 64x64 "
                                          "launch's algorithmic bytes, timed the same way (L2 flushed): the "
                                          "ceiling an event-timed launch of this size can show"}}
    if all(fused):
        # no standalone transform launch in the step: nothing to time, so no number
        tq_roof.update({"achieved": None, "frac": None, "tflops": None})
    if any(fused):
        tq_roof["note"] = ("the transforms of " + ", ".join(L["lin"].name for i, L in enumerate(layers) if fused[i])
                           + " run inside their fused decode launch (roofline) and are not counted here")
    if fig6 is not None:
        # the GEMMs back to back in the step (the INT4 step: codes already in HBM, PDL overlap
        # included), beside the contract's per-launch event timing above
        t4 = fig6["int4_gemm_only_step_ms"] * 1e-3
        g_plain = sum(gemm_min_bytes(T, L["lin"]) for L in layers)
        if decode:
            ach = g_plain / t4 / 1e9
            roof["in_step"] = {"achieved": round(ach, 1), "frac": round(ach / pk["hbm_gbs"], 4), "unit": "GB/s",
                               "per": "compulsory GEMM bytes of the step / the INT4 step (all GEMMs back to back)"}
        else:
            ach = g_ops / t4 / 1e12
            roof["in_step"] = {"achieved": round(ach, 1), "frac": round(ach / int8_peak, 4), "unit": "TOPS",
                               "per": "sum of 2TNK / the INT4 step (all GEMMs back to back)"}
        if not all(fused):
            tq_roof["in_step"] = {"achieved": fig6["in_step_tq_gbs"],
                                  "frac": round(fig6["in_step_tq_gbs"] / pk["hbm_gbs"], 4),
                                  "per": "sum of algorithmic bytes / sum of the transforms' in-step marginal "
                                         "costs (fig6_transform_overhead)"}
    if rank == 0:
        out = {
            "metric": ("decode" if decode else "prefill")
                      + " tokens/s, FlatQuant W4A4 layer linears (transform+quant -> W4A4 GEMM)",
            "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "fp16 in / int4 x int4 -> int32 / fp16 out",
            "data": "synthetic (seeded Gaussian + channel outliers + pivot token; random-init weights)",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "tokens_per_gpu": T, "tokens_total": total_T,
                       "linears": [f"{L['lin'].name} {L['lin'].K}({L['lin'].n1}x{L['lin'].n2})->{L['lin'].N}"
                                   for L in layers],
                       "alpha": args.alpha, "parallelism": f"token-shard x{world} ({scaling} scaling)",
                       "l2": "flushed (256 MiB write then read) before every timed step; flush untimed"},
            "per_gpu": {"value": round(value / world, 1), "unit": "tokens/s"},
            "gpus_active": 1 if rank_lines is None else len({r["pci"] for r in rank_lines}),
            "roofline": roof,
            "tq_roofline": tq_roof,
            "time_share": {"transform_quant": round(tq_ms / ms_per_step, 4), "gemm": round(gemm_ms / ms_per_step, 4),
                           "note": "shares of the serialised per-kernel times (pass 2) relative to the step span (pass 1)"},
            "kernels": kernels,
            "fig6_transform_overhead": fig6,
            "fp16_baseline": fp16,
            "kv_cache_quant": kv,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "host_wall_s_timed_pass": round(wall_s, 3),
        }
        if rank_lines is not None:
            out["ranks"] = rank_lines
        if verify is not None:
            out["verify_allgather"] = verify
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def timed_ms(torch, stream, flush_l2, fn, reps):
    """mean event-timed duration (ms) of fn over reps runs, L2 flushed before each"""
    for _ in range(3):
        fn()
    tot = 0.0
    for _ in range(reps):
        flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps


def int8_peak_tops(pk, peak_src):
    """INT8 dense denominator per the bench contract: the measured bf16 peak (MEASURED_PEAKS.json)
    x the guide's nominal int8/bf16 ratio 2.  The own measurements committed in
    profiles/int8_peak.json (a tcgen05 kind::i8 issue loop on all SMs; cuBLASLt int8 8192^3)
    are reported beside it as alternative denominators."""
    peak = pk["bf16_tflops"] * INT8_PER_BF16
    src = f"{peak_src}: bf16 {pk['bf16_tflops']} TF/s x nominal int8/bf16 ratio 2"
    alt = None
    path = os.path.join(ROOT, "profiles", "int8_peak.json")
    if os.path.exists(path):
        d = json.load(open(path))
        alt = {"tcgen05_issue_loop_tops": d.get("int8_tops"), "cublaslt_int8_8192_tops": d.get("cublaslt_int_mm_8192_tops"),
               "source": "profiles/int8_peak.json (scripts/int8_peak.py)"}
    return peak, src, alt


# ------------------------------------------------------------------------ reference arm
def run_reference(args):
    """Reference arm for this tier: the float64 oracle, timed as it stands on the host cores, on a
    bounded token sample per step (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    cfg = synth.config(args.config)
    sample = 32
    prepared = []
    for lin in cfg["linears"]:
        x = synth.activations(sample, lin.K, seed=1000, tag=lin.name)
        p1 = synth.well_conditioned(lin.n1, seed=0, tag=lin.name + "/p1")
        p2 = synth.well_conditioned(lin.n2, seed=0, tag=lin.name + "/p2")
        w = synth.weights(lin.N, lin.K, seed=0, tag=lin.name)
        qw, sw, _ = O.prepare_weight(w, p1, p2, 1.0)
        prepared.append((x, p1, p2, qw, sw))

    def step():
        for x, p1, p2, qw, sw in prepared:
            qa, sa, _ = O.transform_quant(x, p1, p2, args.alpha)
            O.dequant(O.int_gemm(qa, qw), sa, sw)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    value = sample * args.steps / el
    desc = f"{sample} tokens per step through all {args.config} linears (float64 oracle)"
    print(json.dumps({
        "impl": "reference",
        "metric": ("decode" if cfg["T"] <= 64 else "prefill")
                  + " tokens/s, FlatQuant W4A4 layer linears (transform+quant -> W4A4 GEMM)",
        "value": round(value, 2), "unit": "tokens/s", "n_gpus": int(os.environ.get("WORLD_SIZE", str(args.gpus))),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(el / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong" if args.config in STRONG else "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"{args.config}: {cfg['desc']}", "sample_tokens_per_step": sample},
        "cpu_baseline": {"value": round(value, 2), "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": desc,
                         "nproc": os.cpu_count(), "cpu_model": cpu_model()},
        "e2e": {"value": round(value, 2), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    a = parse()
    launch_or_check_world(a)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
