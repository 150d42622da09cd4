import sys, numpy as np
sys.path.insert(0, '.')
import paper_2407_16559_b200 as agk
from oracle import oracle as O
from tests.helpers import factors, rel_max_diff
P = O.Oracle('port'); F = O.Oracle('port_fma'); Q = O.Oracle('port_pad2')
u, v = factors('brownian2', 4096); md = O.Model(u, v, 1, [(1, 1.0)], 0)
ws = agk.RhsWorkspace(agk.Model(u, v, 1, [(1, 1.0)], 0))
n0 = np.zeros(4096)
st = 0
g = agk.run(ws, agk.SimulationConfig(agk.StepControl(stepper=st, tol=1e-6), 50.0, n0, record=0, records_capacity=100000))
w = P.run(md, n0, O.Control(stepper=st, tol=1e-6), 50.0, record=0, records_capacity=100000)
print('counts', (g.total_rhs_evals, g.total_accepted, g.total_rejects), (w['total_rhs_evals'], w['total_accepted'], w['total_rejects']))
for q in list(range(0, len(g.records), max(1, len(g.records)//12))) + [len(g.records)-1]:
    a, b = g.records[q], w['records'][q]
    print(q, 't %.6f %.6f' % (a['t'], b['t']), 'dN %.2e' % ((a['density']-b['density'])/max(abs(b['density']),1e-300)), 'rej', a['rejects'], b['rejects'])
# RHS bias on the final oracle state
n = w['final_state']
sg = agk.eval_rhs(ws, n); sr = P.eval_rhs(md, n); sf = F.eval_rhs(md, n); sq = Q.eval_rhs(md, n)
print('sum S', sr.sum(), 'gpu-ref', (sg - sr).sum(), 'fma-ref', (sf - sr).sum(), 'pad2-ref', (sq - sr).sum())
print('normwise', rel_max_diff(sg, sr), rel_max_diff(sf, sr), rel_max_diff(sq, sr))
tail = slice(3000, 4096)
print('tail |diff| gpu', np.abs(sg - sr)[tail].mean(), 'pad2', np.abs(sq - sr)[tail].mean(), 'tail |S|', np.abs(sr[tail]).mean())
