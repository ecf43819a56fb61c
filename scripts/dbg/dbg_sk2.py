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
nm, nn, nkb = 8, 22, 32
for tile in range(nm * nn):
    mb, nb = tile % nm, tile // nm
    rows = np.arange(mb * 256, (mb + 1) * 256); cols = np.arange(nb * 192, min((nb + 1) * 192, N))
    ref_blk = qa[rows].astype(np.int64) @ qw[cols].astype(np.int64).T
    b = got[np.ix_(rows, cols)] != ref_blk
    if not b.any():
        continue
    br = np.where(b.any(1))[0]
    print(f"tile {tile} (mb {mb}, nb {nb}): bad rows {br.min()}..{br.max()} ({len(br)}), bad cols/row {b.sum(1).max()}")
    r = rows[br[0]]
    g = got[r, cols]
    parts = np.stack([qa[r, k*128:(k+1)*128].astype(np.int64) @ qw[cols, k*128:(k+1)*128].astype(np.int64).T for k in range(nkb)])
    pre = np.concatenate([np.zeros((1, len(cols)), np.int64), np.cumsum(parts, 0)])
    found = [(a, c) for a in range(nkb) for c in range(a + 1, nkb + 1) if np.array_equal(g, pre[c] - pre[a])]
    print("   got == sum over kb in", found[:4])
    # does got equal another tile's correct values (same in-tile row)?
    for t2 in []:
        mb2, nb2 = t2 % nm, t2 // nm
        r2 = mb2 * 256 + br[0]; c2 = np.arange(nb2 * 192, min((nb2 + 1) * 192, N))
        if len(c2) == len(cols):
            v2 = qa[r2].astype(np.int64) @ qw[c2].astype(np.int64).T
            if np.array_equal(v2, g):
                print("   got == correct values of tile", t2)
    pass
