# small-shape runs of every kernel family for compute-sanitizer (plain, then the tcgen05 tail
# split forced on, then graph-replayed measurements)
import os
import sys
sys.path.insert(0, '.')
import torch
from paper_1909_10616_b200 import tiletune as tt
dev = torch.device('cuda:0')
for fam, n, cfgs in [(1, 128, [((2, 2, 8, 4), (16, 8), (2, 2, 4, 8)), ((128, 1, 1, 1), (128, 1), (128, 1, 1, 1)), ((1, 4, 4, 8), (4, 32), (2, 2, 8, 4)),
                             ((2, 4, 4, 4), (1, 128), (2, 4, 2, 8)), ((2, 2, 8, 4), (2, 64), (2, 4, 4, 4))]),   # fixed-BK instances
                     (3, 512, [((4, 1, 1, 128), (8, 64), (4, 1, 1, 128)), ((1, 2, 2, 128), (8, 64), (2, 1, 1, 256)), ((2, 2, 1, 128), (32, 16), (16, 1, 1, 32))]),
                     (2, 256, [((2, 1, 1, 128), (8, 32), (2, 1, 1, 128)), ((1, 2, 1, 128), (32, 8), (1, 1, 1, 256))])]:
    dt = torch.bfloat16 if fam == 3 else torch.float32
    A = torch.randn(n, n, device=dev).to(dt)
    B = torch.randn(n, n, device=dev).to(dt)
    C = torch.empty(n, n, device=dev)
    for s in cfgs:
        tt.gemm(A, B, C, fam, s)
        torch.cuda.synchronize()
        ref = A.float() @ B.float()
        print(fam, s, float((C - ref).abs().max() / ref.abs().max()))
os.environ["TT_TAIL_SPLIT"] = "2"        # every UMMA config with tiles % clusters != 0 splits
for fam, n, cfgs in [(3, 512, [((4, 1, 1, 128), (8, 64), (4, 1, 1, 128)), ((2, 2, 1, 128), (32, 16), (16, 1, 1, 32))]),
                     (2, 256, [((2, 1, 1, 128), (8, 32), (2, 1, 1, 128))])]:
    dt = torch.bfloat16 if fam == 3 else torch.float32
    A = torch.randn(n, n, device=dev).to(dt)
    B = torch.randn(n, n, device=dev).to(dt)
    C = torch.empty(n, n, device=dev)
    for s in cfgs:
        info = tt.binding(tt.make_space(n, n, n, family=fam), s)
        for _ in range(2):
            tt.gemm(A, B, C, fam, s)
        torch.cuda.synchronize()
        ref = A.float() @ B.float()
        print("split", info.split_tiles, fam, s, float((C - ref).abs().max() / ref.abs().max()))
# A-multicast clusters (n1 = 2), plain and split
for cfg in [((2, 2, 1, 128), (4, 128), (1, 2, 1, 256)), ((4, 1, 1, 128), (4, 128), (2, 2, 1, 128))]:
    A = torch.randn(512, 512, device=dev).to(torch.bfloat16)
    B = torch.randn(512, 512, device=dev).to(torch.bfloat16)
    C = torch.empty(512, 512, device=dev)
    tt.gemm(A, B, C, 3, cfg)
    torch.cuda.synchronize()
    ref = A.float() @ B.float()
    print("multicast", cfg, float((C - ref).abs().max() / ref.abs().max()))
# round 2 default split shape: the last full wave + remainder by stream-K (forced at small sizes)
os.environ["TT_TAIL_SPLIT"] = "4"
for fam, M, N, K, cfg in [(3, 2048, 4096, 256, ((8, 2, 1, 128), (2, 128), (16, 1, 1, 256))),
                          (3, 2048, 2048, 256, ((16, 1, 1, 128), (4, 64), (32, 1, 1, 64)))]:
    A = torch.randn(M, K, device=dev).to(torch.bfloat16)
    B = torch.randn(K, N, device=dev).to(torch.bfloat16)
    C = torch.empty(M, N, device=dev)
    info = tt.binding(tt.make_space(M, N, K, family=fam), cfg)
    for _ in range(2):
        tt.gemm(A, B, C, fam, cfg)
    torch.cuda.synchronize()
    ref = A.float() @ B.float()
    print("wave+remainder split", info.split_tiles, info.split_workers, cfg, float((C - ref).abs().max() / ref.abs().max()))
del os.environ["TT_TAIL_SPLIT"]
ctx = tt.Context(0)
smp = ctx.measure(tt.make_space(512, 512, 512, family=3), ((4, 1, 1, 128), (8, 64), (4, 1, 1, 128)),
                  tt.measure_opts(repeats=2))
print("graph measure ok", smp.graph_nodes, smp.number)
res = tt.gbfs_search(128, 128, 128, 8, tt.search_opts(family=1, seed=0, measure={"repeats": 2}), ctx=ctx)
print("search ok", res.evals)
