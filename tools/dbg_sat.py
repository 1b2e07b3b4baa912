import json, sys
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
gold = json.load(open('tests/golden/counts.json')); plans = json.load(open('tests/golden/plans.json'))
gg = gold['graphs']['er40']; p = plans['sat']
g = mb.DataGraph.from_edges(gg['n'], gg['edges']); qp = mb.QueryPlan(p['k'], p['edges'])
print(mb.count_colorful(g, qp, mb.random_coloring(g, p['k'], 1)))
