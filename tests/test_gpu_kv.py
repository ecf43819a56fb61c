"""GPU parity of the KV-cache quantization kernel (fq_kv_quant) against
the float64 oracle (oracle.kv_quant): per-head transform y = k P_h and
group-wise asymmetric INT4 with one group per head vector (R19, R20)."""
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


def np_of(t):
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        t = t.float()
    return t.numpy()


def kv_inputs(R, D, seed, tdtype, p="orth"):
    # keys: Gaussian head vectors with a few outlier channels (keys are the
    # sensitive side); R = tokens x heads rows
    kv = torch.from_numpy(synth.activations(R, D, seed=seed, tag="kv", dtype=np.float32,
                                            pivot_channels=0, outlier_scale=20.0)).to(tdtype)
    if p == "orth":
        ph = synth.well_conditioned(D, seed=seed, tag="p_h", dtype=np.float32)
    elif p == "identity":
        ph = np.eye(D, dtype=np.float32)
    else:
        ph = synth.hadamard(D).astype(np.float32) / np.sqrt(D)
    return kv, torch.from_numpy(ph).to(tdtype)


def run_and_check(kv, ph, alpha, label):
    q, s, z = fq.kv_quant(kv.to(DEV), ph.to(DEV), alpha)
    torch.cuda.synchronize()
    qo, so, zo, yo = O.kv_quant(kv.float().numpy(), ph.float().numpy(), alpha)
    return parity.check_asym(np_of(q), np_of(s), np_of(z), yo, alpha, qo, so, zo, label=label)


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("R", [1, 127, 128, 1000, 4133])         # ragged tails, several tiles
@pytest.mark.parametrize("tdtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("alpha", [1.0, 0.95])
def test_kv_quant_vs_oracle(D, R, tdtype, alpha):
    kv, ph = kv_inputs(R, D, seed=R + D, tdtype=tdtype)
    run_and_check(kv, ph, alpha, f"kv D={D} R={R} {tdtype} a={alpha}")


@pytest.mark.parametrize("p", ["identity", "hadamard"])
def test_kv_quant_special_transforms(p):
    """Values (P = I) quantize the raw head vectors; a normalised Hadamard P_h."""
    kv, ph = kv_inputs(777, 128, seed=4, tdtype=torch.float16, p=p)
    run_and_check(kv, ph, 1.0, f"kv {p}")


def test_kv_quant_strided_rows_and_degenerate_groups():
    """Row stride > head_dim (a [T, H*D] cache viewed one head at a time is passed as ldkv), an
    all-zero head vector (s = 1, z = 0 -> stored z - 8 = -8, codes 8 - 8 = 0) and one-signed
    groups (zero point at the end of the range)."""
    R, D, H = 300, 128, 4
    base, ph = kv_inputs(R, D * H, seed=9, tdtype=torch.float16, p="identity")
    ph = torch.from_numpy(synth.well_conditioned(D, seed=9, tag="p_h", dtype=np.float32)).half()
    base[5] = 0
    base[7] = base[7].abs()
    base[8] = -base[8].abs()
    bd = base.to(DEV)
    for h in (0, 3):
        view = bd[:, h * D:(h + 1) * D]                      # stride(0) = H*D
        q, s, z = fq.kv_quant(view, ph.to(DEV), 1.0)
        torch.cuda.synchronize()
        qo, so, zo, yo = O.kv_quant(base[:, h * D:(h + 1) * D].float().numpy(), ph.float().numpy(), 1.0)
        parity.check_asym(np_of(q), np_of(s), np_of(z), yo, 1.0, qo, so, zo, label=f"strided h={h}")
        assert np_of(z)[5] == -8 and np_of(s)[5] == 1.0 and np.all(np_of(q)[5] == 0x88)


def test_kv_quant_full_size_sampled():
    """LLaMA-3-8B prefill KV at C3 scale (T = 16384 tokens x 8 KV heads x 128), the launch the
    library issues for the whole cache; sampled head vectors recomputed by the oracle."""
    T, H, D = 16384, 8, 128
    R = T * H
    kv, ph = kv_inputs(R, D, seed=21, tdtype=torch.float16)
    q, s, z = fq.kv_quant(kv.to(DEV), ph.to(DEV), 0.95)
    torch.cuda.synchronize()
    g = np.random.default_rng(0)
    rows = np.concatenate([np.arange(256), g.choice(R, 768, replace=False)])
    qo, so, zo, yo = O.kv_quant(kv[rows].float().numpy(), ph.float().numpy(), 0.95)
    parity.check_asym(np_of(q)[rows], np_of(s)[rows], np_of(z)[rows], yo, 0.95, qo, so, zo, label="kv full")
