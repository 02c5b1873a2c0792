import faulthandler, sys, time, json
faulthandler.dump_traceback_later(60, exit=True)
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from conftest import space_text
from oracle import gp, run, space as S
from parity_util import observed
from paper_2603_11603_b200 import autoscout as A
doc = json.loads(space_text("C4"))
o = S.load_space(doc)
t=time.time(); raws, costs = observed(o, 256, 0); print("observed", time.time()-t, flush=True)
t=time.time(); sp = A.Space(doc, 0); print("space", time.time()-t, flush=True)
t=time.time(); sp.observe(raws, costs); print("observe", time.time()-t, flush=True)
fit = run.observed_fit(o, raws, costs)
d = len(o.features)
hyp = np.array([gp.ml2_candidate(o, 5, h, gp.lengthscales(o), fit.sf2, fit.sn2) for h in range(48)])
t=time.time(); got = sp.gp_lml(hyp); print("lml", time.time()-t, got[:3], flush=True)
