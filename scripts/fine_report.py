"""Report of scripts/fine_trace.sh: mean sub-phase k-cycles per iteration."""
import json
import sys

import numpy as np

names = ['start', '-', 'spmv', 'send n', 'wait mbB', 'scalars', 'own-upd+partials',
         'halo+sync', '-', '-', '-', '-', 'C:start->partials in', 'C:sum+exchange']
recs = [json.loads(ln) for ln in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/fine.jsonl')]
for two in (0, 1):
    rs = [d for d in recs if d['two'] == two]
    if not rs:
        continue
    cs = rs[0]['cs']
    F = np.array([np.array(d['fine'], dtype=np.float64).reshape(-1, 16) / d['iters'] / 1e3 for d in rs])
    print('two', two, 'us/it', round(float(np.median([d['ms'] * 1e3 / d['iters'] for d in rs])), 3),
          'C', F.shape[1])
    Fm = F.mean(0)
    for i, n in enumerate(names):
        if n == '-':
            continue
        col = Fm[::cs, i] if i >= 12 else Fm[:, i]
        print('  %-15s mean %.3f min %.3f max %.3f' % (n, col.mean(), col.min(), col.max()))
    print('  sum(0..11)', round(float(Fm[:, :12].sum(1).mean()), 3))
