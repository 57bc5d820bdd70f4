"""The C ABI holds no device state (include/s24.h, "Conventions"): the GEMMs
distribute their tiles through cluster launch control, not through library
counters. A captured step replayed on one stream while thousands of eager
GEMMs run on another stream must give bit-identical results -- with the
round-1 pool of 4096 scheduler counters, launch 4097 shared a counter slot
with the graph's GEMMs."""

import pytest
import torch

import paper_2503_16672_b200 as s24
from paper_2503_16672_b200 import _lib
from oracle import srelu24_np as O

pytestmark = pytest.mark.gpu


def test_graph_replay_alongside_many_eager_gemms():
    n, d, h = 2048, 512, 2048
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.9, seed=21)
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    step = s24.FfnStepGraph(p, s24.RECIPE, n)
    step.x.copy_(torch.from_numpy(x).cuda().bfloat16())
    step.dy.copy_(torch.from_numpy(dy).cuda().bfloat16())
    step.replay()
    torch.cuda.synchronize()
    ref = [t.clone() for t in (step.out, step.d_x, step.d_w1, step.d_w2)]

    # eager GEMMs (dense and 2:4) on a second stream while the graph replays
    M, N, K = 512, 256, 512
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    a_sp, _, _ = s24.sparsify_token_wise(torch.randn(M, K, device="cuda"))
    D = torch.empty(M, N, device="cuda")
    want_dense = A.float() @ B.float()
    other = torch.cuda.Stream()
    launches = 0
    with torch.cuda.stream(other):
        for i in range(4400):
            if i % 2:
                _lib.call("s24_gemm", A.data_ptr(), 0, K, B.data_ptr(), 1, N, M, N, K, D.data_ptr(), 0, N, None, 0,
                          -1, None, other.cuda_stream)
            else:
                _lib.call("s24_spmm", a_sp.data.data_ptr(), a_sp.meta_hw.data_ptr(), B.data_ptr(), 1, N, M, N, K,
                          D.data_ptr(), 0, N, None, 0, -1, None, 0, other.cuda_stream)
            launches += 1
            if i % 400 == 0:
                step.replay()  # (current stream: runs concurrently with `other`)
    for _ in range(3):
        step.replay()
    torch.cuda.synchronize()
    assert launches == 4400
    for got, want in zip((step.out, step.d_x, step.d_w1, step.d_w2), ref):
        assert torch.equal(got, want)
    # the last eager launch was a dense GEMM: its result is intact too
    assert float((D - want_dense).norm() / want_dense.norm()) < 1e-5
