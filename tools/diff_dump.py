import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle'); sys.path.insert(0, '/root/repo/tools')
import numpy as np
import oracle
from paper_2309_00558_b200 import compiler as cc
import dump_gpu
kind = sys.argv[1]
batch = cc.Batch(dump_gpu.make(kind))
want = oracle.run_batch(batch)
got = dict(np.load(f'/root/repo/gpurun_out/dump_{kind}.npz'))
for r in range(len(batch)):
    s = batch.runs[r]; W, F, G = int(s['windows']), int(s['n_funcs']), int(s['n_nodes'])
    fo, go, lo = int(s['fn_row_off']), int(s['gpu_row_off']), int(s['glob_row_off'])
    for w in range(W):
        a = got['fn_rows'][fo + w*F: fo + (w+1)*F]; b = want['fn_rows'][fo + w*F: fo + (w+1)*F]
        c = got['gpu_rows'][go + w*G: go + (w+1)*G]; d = want['gpu_rows'][go + w*G: go + (w+1)*G]
        e = got['glob_rows'][lo + w]; f = want['glob_rows'][lo + w]
        if not (np.array_equal(a, b) and np.array_equal(c, d) and e == f):
            print('run', r, 'policy', batch.images[r].policy, 'window', w)
            print(' glob got', e, 'want', f)
            for i in range(F):
                if a[i] != b[i]: print(' fn', i, batch.images[r].fids[i], 'got', a[i], 'want', b[i])
            for i in range(G):
                if c[i] != d[i]: print(' gpu', i, 'got', c[i], 'want', d[i])
            break
print('status got', got['status'][['code','token_grants','scale_decisions','placement_attempts']][:8])
print('status want', want['status'][['code','token_grants','scale_decisions','placement_attempts']][:8])
