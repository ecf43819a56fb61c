import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2410_09426_b200 as fq
import oracle as O, synth
T, N, K = 2048, 4096, 4096
qa = synth.random_codes(T, K, seed=T, tag="qa"); qw = synth.random_codes(N, K, seed=N, tag="qw")
acc = fq.w4a4_gemm_i32(torch.from_numpy(O.pack_int4(qa)).cuda(), torch.from_numpy(O.pack_int4(qw)).cuda())
torch.cuda.synchronize()
got = acc.cpu().numpy().astype(np.int64)
ref = O.int_gemm(qa, qw)
nm, nn, nkb = 8, 22, 32
shown = 0
for tile in range(nm * nn):
    mb, nb = tile % nm, tile // nm
    rows = np.arange(mb * 256, (mb + 1) * 256); cols = np.arange(nb * 192, min((nb + 1) * 192, N))
    b = got[np.ix_(rows, cols)] != ref[np.ix_(rows, cols)]
    if not b.any():
        continue
    br = np.where(b.any(1))[0]
    r = rows[br[0]]
    g = got[r, cols]
    # candidates: K-range partial sums of the SAME row/cols
    parts = np.stack([qa[r, k*128:(k+1)*128].astype(np.int64) @ qw[cols, k*128:(k+1)*128].astype(np.int64).T for k in range(nkb)])
    pre = np.concatenate([np.zeros((1, len(cols)), np.int64), np.cumsum(parts, 0)])
    rng = [(a, c) for a in range(nkb) for c in range(a + 1, nkb + 1) if np.array_equal(g, pre[c] - pre[a])]
    # candidate: full result of another row (same cols) -> row mixup in TMEM lanes
    other = [rr for rr in range(T) if np.array_equal(g, ref[rr, cols])]
    # candidate: sum of own full + partial of some range (double counted)
    dbl = [(a, c) for a in range(nkb) for c in range(a + 1, nkb + 1) if np.array_equal(g - ref[r, cols], pre[c] - pre[a])]
    print(f"tile {tile}: bad rows {list(br[:6])}... n={len(br)}; row {r}: partial-range match {rng[:3]}, other-row match {other[:3]}, own+range {dbl[:3]}")
    shown += 1
    if shown >= 6:
        break
