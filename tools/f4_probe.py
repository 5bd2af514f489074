import numpy as np, torch, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle, paper_2112_10591_b200 as ieds
from test_oracle_pins import _square_sequence
dev = torch.device('cuda', 0)
for (W, H, v, L) in ((256, 192, 1, 3), (384, 192, 8, 3), (256, 192, 1, 1)):
    seq = _square_sequence(W, H, v, 10)
    fo = oracle.FlowOracle(W, H, levels=L)
    fe = ieds.FlowEstimator(W, H, levels=L, device=0)
    for k, (S, E) in enumerate(seq):
        S32 = S.astype(np.float32)
        Fo = fo.step(S32.astype(np.float64))
        Fg, vg = fe.step(torch.from_numpy(S32).to(dev))
        torch.cuda.synchronize()
        Fg = Fg.cpu().numpy().astype(np.float64)
        d = np.abs(Fg - Fo)
        print(W, v, L, k, 'max', d.max(), 'mean', d.mean(), 'on E', d[E].max(), 'Fmax', np.abs(Fo).max().round(2))
    fe.close()
