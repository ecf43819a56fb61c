"""tcgen05.mma kind::i8 issue-rate probe (instrumented build): chip-wide TOPS of back-to-back MMAs
on garbage operands for A-in-TMEM vs A-in-smem, CTA pair vs single CTA, N in {128,192,256}."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FQ_TRACE_LIB"] = "1"
import paper_2410_09426_b200 as fq  # noqa: E402
import torch  # noqa: E402,F401

lib = fq.load()
out = (ctypes.c_ulonglong * 2)()
for pair in (1, 0):
    for ts in (1, 0):
        for n in (128, 192, 256):
            ctas = 148
            e = lib.fq_debug_mma_probe(pair | (ts << 1), n, 2000, ctas, out)
            if e != 0:
                print("error", e, pair, ts, n)
                continue
            ns, mmas = out[0], out[1]
            m = 256 if pair else 128
            units = ctas // 2 if pair else ctas
            tops = 2.0 * m * n * 32 * mmas * units / (ns * 1e-9) / 1e12
            cyc = ns * 1.9 / mmas
            print(f"pair={pair} A_in_TMEM={ts} N={n}: {ns / mmas:7.1f} ns/MMA (~{cyc:6.1f} cyc @1.9GHz) -> {tops:7.1f} TOPS chip")
