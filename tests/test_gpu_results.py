"""SURVEY 8(d) result record: one JSON line per (config, linear) with the shape, the transform and
GEMM timings and roofline fractions, per-linear tokens/s against cuBLAS fp16, and the parity
statistics of that linear on sampled tokens (the oracle recomputes exactly those rows).  Written to
gpurun_out/results.jsonl (the record is a by-product; the test asserts the north_star bars).

Timing: L2 write-flushed then read-flushed before every timed launch, CUDA events on the
launching stream, mean of the launches (event ticks are coarse on this part).  t_tq / t_gemm time
the two kernels separately (serialised); t_linear times fq_flatquant_linear, the whole linear as a
user calls it (two kernels overlapped through PDL, or one fused launch at decode sizes)."""
import json
import os
import time

import numpy as np
import pytest
import torch

import oracle as O
import synth
from tests import parity

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2410_09426_b200 as fq
    DEV = torch.device("cuda:0")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HBM_SPEC_GBS, INT8_SPEC_TOPS, F16_SPEC_TFLOPS = 8000.0, 4500.0, 2250.0


def _peaks():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        pk = json.load(f)
    return float(pk["hbm_gbs"]), 2.0 * float(pk["bf16_tflops"])


def _timed(fn, flush, iters=10):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        flush.sum()
        torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return sum(ts) / len(ts)


def _rows(T, n_sample, seed=0):
    if T <= n_sample:
        return np.arange(T)
    g = np.random.default_rng(seed)
    half = n_sample // 2
    return np.unique(np.concatenate([np.arange(half), g.choice(np.arange(half, T), n_sample - half, replace=False)]))


def test_result_records():
    hbm_meas, int8_meas = _peaks()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=DEV)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    out = open(os.path.join(ROOT, "gpurun_out", "results.jsonl"), "w")
    alpha, seed = 0.9, 0
    for cfg_name in ("C1", "C2", "C3", "C4", "C5"):
        cfg = synth.config(cfg_name)
        T = cfg["T"]
        n_sample = 64 if cfg_name == "C5" else 256
        for lin in cfg["linears"]:
            n1, n2, N, K = lin.n1, lin.n2, lin.N, lin.K
            x = synth.activations(T, K, seed=seed, tag=lin.name)
            p1 = synth.well_conditioned(n1, seed=seed, tag=lin.name + "/p1")
            p2 = synth.well_conditioned(n2, seed=seed, tag=lin.name + "/p2")
            qw = synth.random_codes(N, K, seed=seed, tag=lin.name + "/qw")
            sw = synth.random_scales(N, seed=seed, tag=lin.name + "/sw")
            xd = torch.from_numpy(x).to(DEV)
            p1d, p2d = torch.from_numpy(p1).to(DEV), torch.from_numpy(p2).to(DEV)
            qwd, swd = torch.from_numpy(O.pack_int4(qw)).to(DEV), torch.from_numpy(sw).to(DEV)
            q = torch.empty((T, K // 2), dtype=torch.uint8, device=DEV)
            s = torch.empty((T,), dtype=torch.float32, device=DEV)
            y = torch.empty((T, N), dtype=torch.float16, device=DEV)
            t_tq = _timed(lambda: fq.fq_transform_quant(xd, n1, n2, p1d, p2d, alpha, q, s), flush)
            t_gemm = _timed(lambda: fq.fq_w4a4_linear(q, s, qwd, swd, y), flush)
            # the whole-linear entry point: both kernels back to back (PDL), or ONE fused launch at
            # decode sizes (K10); its launch count is recorded with it
            n0 = fq.fq_launch_count()
            fq.fq_flatquant_linear(xd, n1, n2, p1d, p2d, alpha, qwd, swd, y, q, s)
            lin_launches = fq.fq_launch_count() - n0
            t_lin = _timed(lambda: fq.fq_flatquant_linear(xd, n1, n2, p1d, p2d, alpha, qwd, swd, y, q, s), flush)
            w16 = torch.randn((N, K), device=DEV, dtype=torch.float16)
            t_fp16 = _timed(lambda: torch.matmul(xd, w16.t()), flush)
            del w16
            # parity on sampled rows (first half of the sample includes the pivot token 0)
            rows = _rows(T, n_sample, seed=1)
            rr = torch.as_tensor(rows, device=DEV)
            qs, ss, ys = fq.transform_f32(xd[rr], n1, n2, p1d, p2d, alpha)
            acc = fq.w4a4_gemm_i32(q[rr], qwd)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            qo, so, yo = O.transform_quant(x[rows], p1, p2, alpha)
            t_ora_tq = time.perf_counter() - t0
            st = parity.check_transform(qs.cpu().numpy(), ss.cpu().numpy(), ys.cpu().numpy(), yo, qo, so,
                                        label=f"{cfg_name} {lin.name}")
            qa_rows = O.unpack_int4(q[rr].cpu().numpy())
            t0 = time.perf_counter()
            acc_o = O.int_gemm(qa_rows, qw)
            t_ora_gemm = time.perf_counter() - t0
            bit_exact = bool(np.array_equal(acc.cpu().numpy().astype(np.int64), acc_o))
            assert bit_exact
            ref = O.w4a4_linear(qo, so, qw, sw.astype(np.float64))
            same = O.w4a4_linear(qa_rows, s[rr].cpu().numpy().astype(np.float64), qw, sw.astype(np.float64))
            ost = parity.check_output(y[rr].float().cpu().numpy(), ref, same, label=f"{cfg_name} {lin.name}")
            tq_bytes = T * (2 * K + K // 2 + 4) + 2 * (n1 * n1 + n2 * n2)
            tq_flops = 2 * T * K * (n1 + n2)
            gemm_ops = 2 * T * N * K
            rec = {
                "config": cfg_name, "linear": lin.name, "T": T, "n": K, "n1": n1, "n2": n2, "N": N, "G": 1, "rank": 0,
                "dtype": "fp16", "alpha": alpha, "seed": seed,
                "t_tq_us": round(t_tq, 2), "tq_bytes": tq_bytes, "tq_gbs": round(tq_bytes / t_tq / 1e3, 1),
                "tq_frac_hbm_spec": round(tq_bytes / t_tq / 1e3 / HBM_SPEC_GBS, 4),
                "tq_frac_hbm_meas": round(tq_bytes / t_tq / 1e3 / hbm_meas, 4),
                "tq_tensor_floor_us": round(tq_flops / (F16_SPEC_TFLOPS * 1e6), 2),
                "t_gemm_us": round(t_gemm, 2), "gemm_ops": gemm_ops, "gemm_tops": round(gemm_ops / t_gemm / 1e6, 1),
                "gemm_frac_int8_meas": round(gemm_ops / t_gemm / 1e6 / int8_meas, 4),
                "gemm_frac_int8_spec": round(gemm_ops / t_gemm / 1e6 / INT8_SPEC_TOPS, 4),
                "tokens_per_s": round(T / ((t_tq + t_gemm) * 1e-6), 1),
                "fp16_tokens_per_s": round(T / (t_fp16 * 1e-6), 1),
                "speedup_vs_fp16": round(t_fp16 / (t_tq + t_gemm), 3),
                "t_linear_us": round(t_lin, 2), "linear_launches": int(lin_launches),
                "linear_tokens_per_s": round(T / (t_lin * 1e-6), 1),
                "linear_speedup_vs_fp16": round(t_fp16 / t_lin, 3),
                "parity_rows": int(len(rows)),
                "code_mismatch_pct": round(100.0 * st["mismatch_frac"], 5),
                "max_tok_rel_y": st.get("y_rel_max"), "y_rel_fro": ost["out_rel_fro"],
                "out_rel_tok_same_codes": ost["out_rel_tok"], "acc_bit_exact": bit_exact,
                "sm_clock_mhz": None, "oracle_threads": int(os.environ.get("OMP_NUM_THREADS", "0")) or os.cpu_count(),
                "oracle_tq_s_sampled": round(t_ora_tq, 3), "oracle_gemm_s_sampled": round(t_ora_gemm, 3),
                "oracle_extrapolated": T > len(rows),
            }
            try:
                import pynvml
                pynvml.nvmlInit()
                rec["sm_clock_mhz"] = pynvml.nvmlDeviceGetClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0),
                                                                    pynvml.NVML_CLOCK_SM)
            except Exception:
                pass
            out.write(json.dumps(rec) + "\n")
            out.flush()
            del xd, q, s, y
            torch.cuda.empty_cache()
    out.close()
