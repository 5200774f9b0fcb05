import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2601_06288_b200.engine import Engine
from paper_2601_06288_b200.sweeps import sweep
for p in sweep("config5"):
    e = Engine(0)
    out = e.run_batch(p.db, p.model, p.space, p.workloads)
    r = out.results
    print(p.model_name, "survivors max/mean", int(r["n_survivors"].max()), float(r["n_survivors"].mean()),
          "over cap", int((r["n_survivors"] > 2048).sum()), "front max", int(r["n_front"].max()))
    worst = np.argsort(-r["n_survivors"])[:5]
    print("  worst", [(p.workloads[i].isl, p.workloads[i].osl, int(r["n_survivors"][i]), int(r["n_front"][i])) for i in worst])
