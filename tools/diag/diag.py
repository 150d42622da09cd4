import sys, json, numpy as np
sys.path.insert(0, '.')
import paper_2407_16559_b200 as agk
from oracle import oracle as O
from tests.helpers import factors, rel_max_diff
P = O.Oracle('port')
# fake controller rkf45 adaptive decay
n = np.array([0.1, 1.0, 0.3])
ws = agk.fake_rhs(agk.RHS_DECAY, 3)
g = agk.advance(ws, n, 1.0, agk.StepControl(stepper=2, mode=1, tau=0.1, tol=1e-3, max_rejects=5))
w = P.advance(n, 1.0, O.Control(stepper=2, mode=1, tau=0.1, tol=1e-3, max_rejects=5), kind=O.RHS_DECAY)
print('GPU', g.status, g.rejects, g.rhs_evals, g.tau_used, g.tau_next, g.error_estimate, g.state)
print('CPU', w['status'], w['rejects'], w['rhs_evals'], w['tau_used'], w['tau_next'], w['error_estimate'], w['state'])
# single rkf45 step on decay
print('rkf45 step', agk.rkf45_step(ws, n, 1.0), P.rk_step(2, n, 1.0, kind=O.RHS_DECAY))
runs = json.load(open('tests/golden/golden_runs.json'))
for name, c in runs.items():
    u, v = factors(c['kind'], c['m'], c['alpha'])
    ws = agk.RhsWorkspace(agk.Model(u, v, c['variant'], [tuple(s) for s in c['sources']], c['lam']))
    n0 = np.zeros(c['m'])
    if c['variant'] != O.SOURCES: n0[0] = 1.0
    ctl = agk.StepControl(stepper=c['stepper'], mode=c['mode'], tau=c['value'] if c['mode'] == 0 else 0.0, tol=c['value'] if c['mode'] == 1 else 1e-6)
    g = agk.run(ws, agk.SimulationConfig(ctl, c['t_end'], n0, snapshot_times=c['snapshots'], record=0, records_capacity=100000))
    print(name, (g.total_rhs_evals, g.total_accepted, g.total_rejects), (c['total_rhs_evals'], c['total_accepted'], c['total_rejects']), rel_max_diff(g.final_state, np.array(c['final_state'])))
    if name == 'agg_const_rkf45_m256':
        md = O.Model(u, v, c['variant'], [], 0.0)
        w = P.run(md, n0, O.Control(stepper=c['stepper'], mode=c['mode'], tol=c['value']), c['t_end'], snapshot_times=c['snapshots'], record=0, records_capacity=100000)
        for a, b in list(zip(g.records, w['records']))[:8]:
            print('  g', a['t'], a['tau'], a['error_estimate'], a['rejects'])
            print('  w', b['t'], b['tau'], b['error_estimate'], b['rejects'])
