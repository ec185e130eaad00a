import sys, json, faulthandler; faulthandler.enable()
sys.path.insert(0, '.')
import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import scenario as S
sc = json.load(open('tests/golden/scenarios.json'))['correlator_like']
ctx = mb.context(workers=2, devices=2, num_gpus=1)
S.register_gather_kernels(ctx, sc)
got, coh = S.run(ctx, sc)
print('ran', coh, {k: v.ravel()[:3] for k, v in got.items()}, flush=True)
ctx.close()
print('closed', flush=True)
