"""Replay a golden scenario as one batch; report the first move whose report differs from the golden."""
import os, sys
import numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from conftest import load_golden
from paper_2603_28674_b200 import engine as E
name = sys.argv[1] if len(sys.argv) > 1 else 'scn_table4_obstacles_1000_5x'
g = load_golden(name)
eng = E.GpuEngine(E.LayoutView.from_any(g))
reps = eng.batch_update((g['ids'], g['rts']))
got = np.array([[r.new_green, r.new_red, r.new_gray, r.unknown_after_heuristic] for r in reps])
exp = g['reports'][:, :4]
bad = np.nonzero((got != exp).any(1))[0]
st_ok = np.array_equal(eng.states(), g['snap_states'][-1])
print(os.environ.get('RGG_GPU_LIB', 'new'), {k: os.environ[k] for k in os.environ if k.startswith('RGG_') and k != 'RGG_GPU_LIB'},
      'n', len(g['ids']), 'bad moves', len(bad), 'first', bad[:5].tolist(), 'states ok', st_ok)
if len(bad):
    i = bad[0]
    print('  move', i, 'obstacle', g['ids'][i], 'got', got[i].tolist(), 'exp', exp[i].tolist())
