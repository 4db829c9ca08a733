import numpy as np, torch, sys
sys.path.insert(0, '.')
import synth
from paper_1909_10616_b200 import tiletune as tt
dev = torch.device('cuda:0')
def run(cfg, A, B, fam=2):
    Ad = torch.from_numpy(A).to(dev); Bd = torch.from_numpy(B).to(dev)
    if fam == 3: Ad, Bd = Ad.bfloat16(), Bd.bfloat16()
    C = torch.full((A.shape[0], B.shape[1]), float('nan'), device=dev)
    tt.gemm(Ad, Bd, C, fam, cfg); torch.cuda.synchronize(); return C.cpu().numpy()
np.set_printoptions(linewidth=200, precision=3)
n = 128
I = np.eye(n, dtype=np.float32)
R = synth.uniform_f32(2, n, n)
# rounded-to-tf32 inputs so conversion mode does not matter
Rt = (R.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
for cfg in [((1,1,1,128),(4,32),(1,1,1,128)), ((1,1,1,128),(16,8),(1,1,1,128)), ((1,1,1,128),(8,16),(8,1,1,16))]:
    C1 = run(cfg, I, Rt)   # tests B path
    C2 = run(cfg, Rt, I)   # tests A path
    print(cfg, 'A=I err', np.abs(C1 - Rt).max(), 'B=I err', np.abs(C2 - Rt).max())
    if np.abs(C1-Rt).max() > 0:
        # find where each C1 row/col comes from
        for i in range(3):
            row = C1[i]
            # match columns
            idx = [np.where(np.all(np.isclose(Rt, row[None,:]), axis=1))[0] for _ in [0]]
            print(' C1 row', i, row[:8], ' Rt row', Rt[i,:8])
        # column mapping: which Rt column equals C1 column j
        mp = []
        for j in range(16):
            m = [k for k in range(n) if np.allclose(C1[:, j], Rt[:, k])]
            mp.append(m[:2])
        print(' colmap', mp)
        rm = []
        for i in range(16):
            m = [k for k in range(n) if np.allclose(C1[i, :], Rt[k, :])]
            rm.append(m[:2])
        print(' rowmap', rm)
    if np.abs(C2-Rt).max() > 0:
        print(' C2 row0', C2[0,:8], 'Rt', Rt[0,:8])
# probe conversion with B low bits set
C = run(((1,1,1,128),(4,32),(1,1,1,128)), I, R)
bits = R.view(np.uint32)
print('conv: exact', np.array_equal(C, R), 'trunc', np.array_equal(C, (bits & np.uint32(0xFFFFE000)).view(np.float32)),
      'rne/rna?', np.abs(C - R).max(), np.abs(C-Rt).max())
