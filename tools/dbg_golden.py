import json, sys
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
gold = json.load(open('tests/golden/counts.json')); plans = json.load(open('tests/golden/plans.json'))
only = sys.argv[1] if len(sys.argv) > 1 else None
for case in gold['cases']:
    if only and case['query'] != only: continue
    gg = gold['graphs'][case['graph']]; p = plans[case['query']]
    g = mb.DataGraph.from_edges(gg['n'], gg['edges']); qp = mb.QueryPlan(p['k'], p['edges'])
    chi = mb.random_coloring(g, p['k'], case['seed'])
    print(case, qp.canonical(), flush=True)
    c = mb.count_colorful(g, qp, chi)
    print('   ->', c, c == case['colorful'], flush=True)
