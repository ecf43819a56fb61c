import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2410_09426_b200 as fq
import oracle as O, synth
T, N, K = 2048, 4096, 4096
qa = synth.random_codes(T, K, seed=T, tag="qa"); qw = synth.random_codes(N, K, seed=N, tag="qw")
qa_d = torch.from_numpy(O.pack_int4(qa)).cuda(); qw_d = torch.from_numpy(O.pack_int4(qw)).cuda()
qa0 = qa_d.clone(); qw0 = qw_d.clone()
print("qa", hex(qa_d.data_ptr()), "qw", hex(qw_d.data_ptr()))
for i in range(3):
    acc = fq.w4a4_gemm_i32(qa_d, qw_d)
    torch.cuda.synchronize()
    print("qa modified:", not torch.equal(qa_d, qa0), "qw modified:", not torch.equal(qw_d, qw0), "acc", hex(acc.data_ptr()))
    ref = O.int_gemm(qa, qw)
    print("bad frac", (acc.cpu().numpy() != ref).mean())
