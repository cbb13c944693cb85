import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle'); sys.path.insert(0, '/root/repo/tests')
from harness import RefCase
from paper_2411_17651_b200.engine import Engine
eng = Engine(0)
for key in sys.argv[1:]:
    c = RefCase(key, '/tmp/psg_probe')
    r = eng.search(c.plans, c.cluster, c.store, c.trace, c.config())
    e = r.entries
    import numpy as np
    it = e['num_iterations'].astype(float)
    print(key, 'avg B overall', r.sum_batch / r.total_iterations, 'max_batch median', np.median(e['max_batch_observed']), 'max', e['max_batch_observed'].max())
    k = int(np.argmax(it)); print('  longest entry', r.encoding(k), 'iters', int(it[k]), 'maxB', int(e['max_batch_observed'][k]))
