import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2410_09426_b200 as fq
import oracle as O, synth
T, N, K = 2048, 4096, 4096
qa = synth.random_codes(T, K, seed=T, tag="qa"); qw = synth.random_codes(N, K, seed=N, tag="qw")
acc = fq.w4a4_gemm_i32(torch.from_numpy(O.pack_int4(qa)).cuda(), torch.from_numpy(O.pack_int4(qw)).cuda())
torch.cuda.synchronize()
ref = O.int_gemm(qa, qw)
got = acc.cpu().numpy().astype(np.int64)
bad = got != ref
print("bad frac", bad.mean())
# per tile (256 x 192)
nm, nn = (T + 255)//256, (N + 191)//192
for tile in range(nm*nn):
    mb, nb = tile % nm, tile // nm
    blk = bad[mb*256:(mb+1)*256, nb*192:(nb+1)*192]
    if blk.any():
        r0 = blk[:128].any(); r1 = blk[128:].any()
        d = (got - ref)[mb*256:(mb+1)*256, nb*192:(nb+1)*192]
        print("tile", tile, "mb", mb, "nb", nb, "rank0 bad", r0, "rank1 bad", r1, "frac", blk.mean(), "diff sample", d[blk][:3], "ref sample", ref[mb*256:(mb+1)*256, nb*192:(nb+1)*192][blk][:3])
# detail: tile 3 and tile 5 bad rows, and whether diff equals +- one k-block's contribution
for tile in (3, 5):
    mb, nb = tile % nm, tile // nm
    rows = np.arange(mb*256, (mb+1)*256); cols = np.arange(nb*192, min((nb+1)*192, N))
    b = bad[np.ix_(rows, cols)]
    badrows = rows[b.any(1)]
    print("tile", tile, "bad rows", badrows.min() - mb*256, "..", badrows.max() - mb*256, "count", len(badrows), "bad cols per row", b.sum(1).max())
    r = badrows[0]; d = (got - ref)[r, cols]
    for kb in range(K // 128):
        part = qa[r, kb*128:(kb+1)*128].astype(np.int64) @ qw[cols, kb*128:(kb+1)*128].astype(np.int64).T
        for sgn in (1, -1):
            if np.array_equal(d, sgn * part):
                print("  diff == ", sgn, "* kblock", kb)
    # cumulative: diff == -(sum of kb < x) ?
    cum = np.zeros_like(d)
    for kb in range(K // 128):
        cum = cum + qa[r, kb*128:(kb+1)*128].astype(np.int64) @ qw[cols, kb*128:(kb+1)*128].astype(np.int64).T
        if np.array_equal(d, -cum) or np.array_equal(d, cum): print("  diff == +-prefix up to kb", kb)
