import json, sys, numpy as np, torch
sys.path.insert(0,'.')
import paper_2208_07678_b200 as fec
cases=json.load(open('tests/golden/spec_examples.json'))['cases']
for c in cases:
    pts=np.array(c['points'],np.float32).reshape(-1,3)
    try:
        lab=fec.cluster(torch.from_numpy(pts).cuda(), c['d_th'], c['min_size'], c['max_size']); torch.cuda.synchronize()
        print('ok', c['name'])
    except Exception as e:
        print('FAIL', c['name'], pts.tolist()[:6], c['d_th']); break
