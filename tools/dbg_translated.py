import sys, numpy as np
sys.path.insert(0, '.')
from oracle.oracle import Oracle
from paper_2103_07414_b200 import mosaic as M
g = dict(np.load('tests/golden/blend_translated.npz'))
polys=[]; o=0
for n in g['npoly']: polys.append(g['polys'][o:o+n]); o+=n
O = Oracle(); ctx = M.Context(0)
for steps in (1, 2):
    cv = M.Canvas(ctx); ocv = O.canvas()
    for k in range(steps):
        st = M.blend_frame(cv, g['frame'], g['anchors'], g['warps'][k], float(g['alpha']), polys[k])
        so = O.blend_frame(ocv, g['frame'], g['anchors'], g['warps'][k], float(g['alpha']), polys[k])
        print(steps, k, st, so)
    col, wt = cv.read(); ocol, owt = ocv.arrays()
    d = np.argwhere(wt != owt)
    print("steps", steps, "ndiff", len(d))
    if len(d):
        print("rows", np.unique(d[:,0])[:20], "cols", np.unique(d[:,1])[:40])
        for (y,x) in d[:10]: print(y, x, wt[y,x], owt[y,x])
