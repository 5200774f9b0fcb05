"""Small driver for ncu captures: one batch of a named sweep (default config5), then one replay.

    ncu --set full -k regex:k_eval -s 1 -c 1 -o gpurun_out/prof python tools/profile_run.py [model] [n_workloads] [sweep]
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2601_06288_b200.engine import Engine  # noqa: E402
from paper_2601_06288_b200.sweeps import sweep  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "gpt-oss-120b"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
sweep_name = sys.argv[3] if len(sys.argv) > 3 else "config5"
part = next(p for p in sweep(sweep_name) if p.model_name == model)
eng = Engine(0)
out = eng.run_batch(part.db, part.model, part.space, part.workloads[:n])
tot = eng.replay(1)
print(f"{model}: {int(out.results['n_enumerated'].sum())} candidates, kernel ms {list(tot.kernel_ms)}")
