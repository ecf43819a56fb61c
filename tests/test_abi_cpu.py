"""The C-ABI library loads on a CPU-only box, exports every symbol include/flatquant.h declares,
and its host-side validation rejects bad arguments before any launch (no GPU needed)."""
import ctypes
import os
import re

import pytest

import oracle as O
import paper_2410_09426_b200 as fq
from paper_2410_09426_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flatquant.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fq_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = fq.load()
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), f"{n} declared in flatquant.h but not exported"
    # the binding covers the same set
    assert set(names) == set(_lib.SIGNATURES)


def test_abi_version_and_status_strings():
    lib = fq.load()
    assert fq.fq_abi_version() == 5
    for s in range(5):
        assert lib.fq_status_string(s).startswith(b"FQ_")
    assert lib.fq_status_string(99) == b"unknown fq_status"


def test_choose_decomposition_matches_oracle_rule():
    for n in list(range(1, 2000)) + [4096, 8192, 11008, 14336, 28672, 57344]:
        assert fq.fq_choose_decomposition(n) == O.choose_decomposition(n)


VP = ctypes.c_void_p
A16 = VP(0x1000)     # aligned fake device pointers: validation must reject before any use
MIS = VP(0x1001)


def tq(**kw):
    args = dict(x=A16, dt=0, T=4, ldx=512, n1=16, n2=32, p1=A16, p2=A16, alpha=1.0, qmode=0, q=A16, s=A16,
                zero=None, stream=None)
    args.update(kw)
    return fq.load().fq_transform_quant(args["x"], args["dt"], args["T"], args["ldx"], args["n1"], args["n2"],
                                        args["p1"], args["p2"], args["alpha"], args["qmode"], args["q"], args["s"],
                                        args["zero"], args["stream"])


def test_transform_quant_validation():
    assert tq(T=0) == _lib.FQ_OK                          # nothing to do, no launch
    assert tq(alpha=0.0) == _lib.FQ_EINVAL
    assert tq(alpha=1.5) == _lib.FQ_EINVAL
    assert tq(alpha=float("nan")) == _lib.FQ_EINVAL
    assert tq(dt=7) == _lib.FQ_EINVAL
    assert tq(qmode=1) == _lib.FQ_EINVAL                  # asymmetric mode needs the zero buffer
    assert tq(qmode=1, T=0, zero=A16) == _lib.FQ_OK
    assert tq(qmode=3) == _lib.FQ_EINVAL
    assert tq(zero=A16) == _lib.FQ_EINVAL                 # symmetric mode takes no zero buffer
    assert tq(x=None) == _lib.FQ_EINVAL
    assert tq(q=None) == _lib.FQ_EINVAL
    assert tq(T=-1) == _lib.FQ_EINVAL
    assert tq(n1=3, n2=5, ldx=16) == _lib.FQ_ESHAPE        # odd n cannot be nibble-packed
    assert tq(ldx=256) == _lib.FQ_ESHAPE                  # ldx < n
    assert tq(ldx=516) == _lib.FQ_ESHAPE                  # row stride not 16-byte multiple
    assert tq(x=MIS) == _lib.FQ_ESHAPE
    assert tq(n1=512, n2=2, ldx=1024) == _lib.FQ_ENOTSUP
    # multiples of 16 with no tensor-core kernel and too large for the CUDA-core kernel's shared
    # memory: rejected up front, not launched
    assert tq(n1=256, n2=256, ldx=65536) == _lib.FQ_ENOTSUP
    assert tq(n1=192, n2=192, ldx=36864) == _lib.FQ_ENOTSUP
    # p2 = NULL means P2 = I (the paper's online P_o (x) I_{d_head}); only (32|64, 128), symmetric
    assert tq(p2=None) == _lib.FQ_ENOTSUP                 # 16 x 32: no P2 = I kernel
    assert tq(p2=None, n1=32, n2=128, ldx=4096, qmode=1, zero=A16) == _lib.FQ_ENOTSUP
    assert tq(p2=None, n1=32, n2=128, ldx=4096, T=0) == _lib.FQ_OK


def gemm(**kw):
    a = dict(qa=A16, sa=A16, za=None, T=8, K=64, qw=A16, sw=A16, cs=None, N=16, y=A16, dt=0, stream=None)
    a.update(kw)
    return fq.load().fq_w4a4_linear(a["qa"], a["sa"], a["za"], a["T"], a["K"], a["qw"], a["sw"], a["cs"], a["N"],
                                    a["y"], a["dt"], a["stream"])


def test_w4a4_linear_validation():
    assert gemm(T=0) == _lib.FQ_OK
    assert gemm(N=0) == _lib.FQ_OK
    assert gemm(K=48) == _lib.FQ_ESHAPE                   # K % 32
    assert gemm(N=12) == _lib.FQ_ESHAPE                   # N % 8
    assert gemm(qa=None) == _lib.FQ_EINVAL
    assert gemm(sa=None) == _lib.FQ_EINVAL
    assert gemm(dt=5) == _lib.FQ_EINVAL
    assert gemm(za=A16) == _lib.FQ_EINVAL                 # zero points without colsum_w
    assert gemm(cs=A16) == _lib.FQ_EINVAL                 # colsum_w without zero points
    assert gemm(za=A16, cs=MIS) == _lib.FQ_ESHAPE
    lib0 = fq.load()
    assert lib0.fq_weight_colsum(None, 4, 64, A16, None) == _lib.FQ_EINVAL
    assert lib0.fq_weight_colsum(A16, 4, 63, A16, None) == _lib.FQ_ESHAPE
    assert lib0.fq_weight_colsum(A16, 0, 64, A16, None) == _lib.FQ_OK
    assert gemm(y=MIS) == _lib.FQ_ESHAPE
    assert gemm(K=262144) == _lib.FQ_ENOTSUP
    # 256 |acc| <= 2^14 K must stay below 2^31 in the widened (16 q) accumulator: K < 131072
    assert gemm(K=131072) == _lib.FQ_ENOTSUP
    assert gemm(K=131072, za=A16, cs=A16) == _lib.FQ_ENOTSUP
    lib = fq.load()
    assert lib.fq_w4a4_gemm_i32(A16, 8, 40, A16, 16, A16, None) == _lib.FQ_ESHAPE
    assert lib.fq_w4a4_gemm_i32(None, 8, 64, A16, 16, A16, None) == _lib.FQ_EINVAL
    assert lib.fq_set_gemm_impl(8) == _lib.FQ_EINVAL and lib.fq_set_gemm_impl(-1) == _lib.FQ_EINVAL


def kvq(**kw):
    a = dict(kv=A16, dt=0, R=8, ld=128, D=128, p=A16, alpha=1.0, q=A16, s=A16, z=A16, stream=None)
    a.update(kw)
    return fq.load().fq_kv_quant(a["kv"], a["dt"], a["R"], a["ld"], a["D"], a["p"], a["alpha"], a["q"], a["s"],
                                 a["z"], a["stream"])


def test_kv_quant_validation():
    assert kvq(R=0) == _lib.FQ_OK
    assert kvq(R=-1) == _lib.FQ_EINVAL
    assert kvq(dt=3) == _lib.FQ_EINVAL
    assert kvq(alpha=0.0) == _lib.FQ_EINVAL
    assert kvq(alpha=float("nan")) == _lib.FQ_EINVAL
    assert kvq(ld=64) == _lib.FQ_EINVAL                   # row stride < head_dim
    for k in ("kv", "p", "q", "s", "z"):
        assert kvq(**{k: None}) == _lib.FQ_EINVAL
    assert kvq(D=96, ld=96) == _lib.FQ_ENOTSUP            # head_dim 64 or 128
    assert kvq(kv=MIS) == _lib.FQ_ESHAPE
    assert kvq(ld=132) == _lib.FQ_ESHAPE                  # row stride not a 16-byte multiple


def test_prepare_weight_validation():
    lib = fq.load()
    ws_need = lib.fq_prepare_weight_workspace_size(64, 64)
    assert ws_need >= 64 * 128 * 8 + 2 * 64 * 64 * 2
    assert lib.fq_prepare_weight_workspace_size(0, 64) == 0 and lib.fq_prepare_weight_workspace_size(64, 512) == 0

    def pw(**kw):
        a = dict(w=A16, dt=0, N=8, ld=4096, n1=64, n2=64, p1=A16, p2=A16, alpha=1.0, qw=A16, sw=A16, cs=None,
                 ws=A16, wsb=ws_need, stream=None)
        a.update(kw)
        return lib.fq_prepare_weight(a["w"], a["dt"], a["N"], a["ld"], a["n1"], a["n2"], a["p1"], a["p2"],
                                     a["alpha"], a["qw"], a["sw"], a["cs"], a["ws"], a["wsb"], a["stream"])
    assert pw(N=0) == _lib.FQ_OK
    assert pw(ws=None) == _lib.FQ_EINVAL
    assert pw(wsb=ws_need - 1) == _lib.FQ_EINVAL
    assert pw(ws=VP(0x1010)) == _lib.FQ_ESHAPE            # workspace must be 256-byte aligned
    assert pw(cs=MIS) == _lib.FQ_ESHAPE
    assert pw(p1=None) == _lib.FQ_EINVAL
    assert pw(alpha=0.0) == _lib.FQ_EINVAL
    assert pw(n1=300, n2=2, ld=600) == _lib.FQ_ENOTSUP
    assert "singular" in lib.fq_status_string(_lib.FQ_ESINGULAR).decode()


def test_gemm_impl_selector_validation():
    assert fq.load().fq_set_gemm_impl(8) == _lib.FQ_EINVAL
    with pytest.raises(fq.FlatQuantError):
        fq.fq_set_gemm_impl(-1)


def test_tq_impl_selector_validation():
    lib = fq.load()
    assert lib.fq_set_tq_impl(3) == _lib.FQ_EINVAL and lib.fq_set_tq_impl(-1) == _lib.FQ_EINVAL
    for impl in (2, 1, 0):
        assert lib.fq_set_tq_impl(impl) == _lib.FQ_OK


def test_product_path_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2410_09426_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle's", ""), f


def test_graft_entry_build_is_consistent():
    """__graft_entry__.build() (the driver's build check) compiles/loads the library and its
    ABI assertion matches the header (cached build: no recompilation when nothing changed)."""
    import __graft_entry__ as g
    g.build()
    assert fq.fq_abi_version() == 5


def test_linear_host_async_validates_before_copying():
    """Every argument check of the hot path runs before the host-buffer entry point enqueues its
    H2D copy (nothing is enqueued on error): bad alpha, N % 8, misaligned scales, negative n1."""
    lib = fq.load()

    def call(**kw):
        a = dict(xh=A16, xd=A16, dt=0, T=4, n1=16, n2=32, p1=A16, p2=A16, alpha=0.9, qw=A16, sw=A16, N=16,
                 yh=A16, yd=A16, ydt=0, q=A16, s=A16)
        a.update(kw)
        return lib.fq_flatquant_linear_host_async(a["xh"], a["xd"], a["dt"], a["T"], a["n1"], a["n2"], a["p1"],
                                                  a["p2"], a["alpha"], a["qw"], a["sw"], a["N"], a["yh"], a["yd"],
                                                  a["ydt"], a["q"], a["s"], None)
    assert call(alpha=1.5) == _lib.FQ_EINVAL
    assert call(N=12) == _lib.FQ_ESHAPE
    assert call(sw=MIS) == _lib.FQ_ESHAPE
    assert call(n1=-3) == _lib.FQ_EINVAL
    assert call(T=0) == _lib.FQ_OK
