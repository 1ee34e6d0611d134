import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2603_28674_b200 import engine as E
g = dict(np.load('tests/golden/scn_quick_smoke.npz'))
print('load', flush=True)
eng = E.GpuEngine(E.LayoutView.from_any(g)); print('created', flush=True)
eng.update_async(g['ids'][:1], g['rts'][:1]); print('enqueued', flush=True)
eng.sync(); print('synced 1', flush=True)
st = eng.last_stats(); print(st, flush=True)
print(eng.states()[:10], flush=True)
