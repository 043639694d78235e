import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2505_05950_b200 as fb
from oracle import oracle as O
dh, di = 4096, int(sys.argv[1])
g,u,d = O.seeded_expert(dh, di, 99); x = O.seeded_input(dh, 100)
q = O.quantize(u, 2, 64); v = O.qgemv_channels(q, dh, x); t = O.calibrate_threshold(np.abs(v), 0.8)
e = fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=g, down=d, threshold=t)
ws = fb.Workspace(dh, di)
xd = torch.from_numpy(x).cuda()
print("start", flush=True)
for outputs in (False, True):
    kw = {}
    if outputs:
        kw = dict(v=torch.empty(di, device='cuda'), mask=torch.empty(di, dtype=torch.uint8, device='cuda'),
                  kept=torch.empty(di, dtype=torch.int32, device='cuda'), n_kept=torch.zeros(1, dtype=torch.int32, device='cuda'))
    y = fb.expert_forward_sparse(e, xd, ws, **kw); torch.cuda.synchronize()
    ref = O.expert_forward_sparse(O.Expert(dh, di, q, g, d, t), x)
    print(di, outputs, 'rel', O.rel_l2(y.cpu().numpy(), ref), flush=True)
