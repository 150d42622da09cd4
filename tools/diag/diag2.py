import sys, json, numpy as np
sys.path.insert(0, '.')
import paper_2407_16559_b200 as agk
from oracle import oracle as O
from tests.helpers import factors, rel_max_diff
P = O.Oracle('port')
def cmp(kind, m, alpha, var, srcs, lam, stepper, tol, t_end, n0):
    u, v = factors(kind, m, alpha)
    ws = agk.RhsWorkspace(agk.Model(u, v, var, srcs, lam))
    md = O.Model(u, v, var, srcs, lam)
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(stepper=stepper, tol=tol), t_end, n0, record=0, records_capacity=100000))
    w = P.run(md, n0, O.Control(stepper=stepper, tol=tol), t_end, record=0, records_capacity=100000)
    print(kind, m, 'counts', (g.total_rhs_evals, g.total_accepted, g.total_rejects), (w['total_rhs_evals'], w['total_accepted'], w['total_rejects']))
    first = None
    errs = []
    for q, (a, b) in enumerate(zip(g.records, w['records'])):
        if a['rejects'] != b['rejects'] and first is None:
            first = q
        if q > 0 and first is None:
            errs.append(abs(a['error_estimate'] / b['error_estimate'] - 1))
            errs_t = abs(a['tau'] / b['tau'] - 1)
    print(' first divergence at record', first, 'of', len(g.records), ' max rel err-estimate diff before', max(errs) if errs else None, 'median', np.median(errs) if errs else None)
    if first:
        for q in range(max(1, first - 2), first + 2):
            a, b = g.records[q], w['records'][q]
            print('  ', q, 'g t=%.17g tau=%.17g err=%.17g rej=%d' % (a['t'], a['tau'], a['error_estimate'], a['rejects']))
            print('  ', q, 'w t=%.17g tau=%.17g err=%.17g rej=%d' % (b['t'], b['tau'], b['error_estimate'], b['rejects']))
    print(' N rel diff', abs(g.records[-1]['density'] / w['records'][-1]['density'] - 1))
cmp('brownian2', 4096, 0.0, 1, [(1, 1.0)], 0.0, 2, 1e-6, 50.0, np.zeros(4096))
cmp('brownian2', 4096, 0.0, 1, [(1, 1.0)], 0.0, 1, 1e-6, 50.0, np.zeros(4096))
n0 = np.zeros(2048); n0[0] = 1
cmp('brownian', 2048, 0.9, 2, [], 0.01, 2, 1e-8, 20.0, n0)
cmp('brownian2', 512, 0.0, 1, [(1, 1.0)], 0.0, 2, 1e-6, 20.0, np.zeros(512))
