import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_cs_0610046_b200 as mm, synth
img = synth.c4(count=2, rows=256, cols=512, nrect=6)
x = torch.from_numpy(img).cuda()
for C0 in (498, 500, 496):
    wr = 512 - C0 + 1
    R, C = 256 - 14, C0
    ox = torch.zeros(2, R, 512, dtype=torch.uint8, device='cuda')
    on = torch.zeros(2, R, 512, dtype=torch.uint8, device='cuda')
    try:
        mm.maxmin_filter_2d(x, 15, 15, out_max=ox[:, :, :C], out_min=on[:, :, :C])
    except Exception as e:
        print(e); continue
    pad = ox[:, :, C:].cpu().numpy()
    nz = np.nonzero(pad)
    print(C0, 'nonzero pad cols', np.unique(nz[2]) + C, 'rows', np.unique(nz[1])[:10], 'count', len(nz[0]))
