import json, sys, subprocess
sys.path.insert(0, '.')
gold = json.load(open('tests/golden/counts.json')); plans = json.load(open('tests/golden/plans.json'))
code = '''
import json, sys
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
gold = json.load(open('tests/golden/counts.json')); plans = json.load(open('tests/golden/plans.json'))
gname, qname, tree = sys.argv[1], sys.argv[2], int(sys.argv[3])
gg = gold['graphs'][gname]; p = plans[qname]
g = mb.DataGraph.from_edges(gg['n'], gg['edges']); qp = mb.QueryPlan(p['k'], p['edges'])
if tree >= 0: qp.use_tree(tree)
try:
    print(qp.canonical(), mb.count_colorful(g, qp, mb.random_coloring(g, p['k'], 1)))
except Exception as e:
    print(qp.canonical(), 'ERR', str(e)[:100])
'''
open('/tmp/one.py','w').write(code)
for gname, qname, tree in [('er40','sat',-1)] + [('er40','sat',t) for t in range(19)] + [('er40','theta',t) for t in range(3)] + [('er40','c5',-1)]:
    r = subprocess.run([sys.executable, '/tmp/one.py', gname, qname, str(tree)], capture_output=True, text=True, env=dict(__import__('os').environ, MB_SYNC_DEBUG='1'))
    print(gname, qname, tree, (r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:220], flush=True)
