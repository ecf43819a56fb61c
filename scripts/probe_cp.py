"""Probe of the hardware INT4 decompression path (instrumented build, fq_probe_cp.cu):
TMA 16U4_ALIGN16B smem image and tcgen05.cp .b8x16.b4x16_p64 TMEM image, compared against
candidate nibble -> byte mappings."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FQ_TRACE_LIB"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_09426_b200 as fq  # noqa: E402

lib = fq.load()
f = lib.fq_debug_cp_probe
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]

rng = np.random.default_rng(0)
packed = rng.integers(0, 256, size=(256, 128), dtype=np.uint8)
nib = np.empty((256, 256), np.int64)
nib[:, 0::2] = packed & 15
nib[:, 1::2] = packed >> 4
pk = torch.from_numpy(packed).cuda()

cands = {
    "n (zero-ext, bits 3:0)": lambda n: n,
    "n<<2 (bits 5:2)": lambda n: n << 2,
    "n<<4 (bits 7:4)": lambda n: n << 4,
    "sext(n) & 0xff": lambda n: (np.where(n >= 8, n - 16, n)) & 0xFF,
    "n ^ 8": lambda n: n ^ 8,
    "(n<<2)^0x20": lambda n: (n << 2) ^ 0x20,
}

for mode in [int(m) for m in (sys.argv[1:] or ['0', '4', '9', '1', '13', '5'])]:
    sd = torch.zeros(2 * 32768, dtype=torch.uint8, device="cuda")
    td = torch.zeros(2 * 128 * 64, dtype=torch.int32, device="cuda")
    e = f(pk.data_ptr(), mode, sd.data_ptr(), td.data_ptr())
    print(f"=== mode {mode} ({['manual lo8', 'tma', 'manual hi8'][mode & 3]}, pair={bool(mode & 4)}) status {e}")
    if e != 0:
        continue
    torch.cuda.synchronize()
    smem = sd.cpu().numpy().reshape(2, 2, 128, 128)   # [cta][half][row][128 B swizzled]
    tm = td.cpu().numpy().view(np.uint8).reshape(2, 128, 256)   # [cta][row][byte]
    for cta in range(2 if mode & 4 else 1):
        rows = slice(cta * 128, cta * 128 + 128)
        if mode & 3 == 1:
            # un-swizzle unit g of row r and show where the 8 packed bytes went
            r = 3
            for g in (0, 1):
                u = smem[cta, 0, r, ((g ^ (r % 8)) * 16):((g ^ (r % 8)) * 16) + 16]
                print(f"  cta{cta} smem row {r} unit {g}: {' '.join(f'{b:02x}' for b in u)}"
                      f"   packed: {' '.join(f'{b:02x}' for b in packed[cta * 128 + r, 8 * g:8 * g + 8])}")
        got = tm[cta]
        exp_n = nib[rows]
        print(f"  cta{cta} tmem row 3 bytes 0-15: {' '.join(f'{b:02x}' for b in got[3, :16])}")
        print(f"  cta{cta} nibbles row 3 0-15:    {' '.join(f'{b:02x}' for b in exp_n[3, :16])}")
        for name, fn in cands.items():
            ok = np.mean(got == fn(exp_n).astype(np.uint8))
            print(f"  cta{cta} match {name:24s}: {ok:.4f}")
