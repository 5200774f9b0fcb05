"""Projected per-rank step time of the config-5 sweep at N = 1, 2, 4, 8 GPUs.

Rank 0's block of every model's workloads (bench.py's sharding) is run alone on
one B200 -- both models' pipelines in flight on their own streams, timed with
CUDA events as bench.py times them -- to show how the fixed sweep divides.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2601_06288_b200.dist import shard_range  # noqa: E402
from paper_2601_06288_b200.engine import Engine  # noqa: E402
from paper_2601_06288_b200.sweeps import sweep  # noqa: E402

parts = sweep("config5")
for world in (1, 2, 4, 8):
    engines, cands = [], 0
    for p in parts:
        lo, hi = shard_range(len(p.workloads), 0, world)
        e = Engine(0)
        out = e.run_batch(p.db, p.model, p.space, p.workloads[lo:hi])
        cands += int(out.results["n_enumerated"].sum())
        engines.append(e)
    streams = [torch.cuda.ExternalStream(e.stream_ptr()) for e in engines]
    cur = torch.cuda.current_stream()
    ts = []
    for it in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        for st in streams:
            st.wait_event(a)
        for e in engines:
            e.replay_async()
        for st in streams:
            d = torch.cuda.Event()
            d.record(st)
            cur.wait_event(d)
        b.record(cur)
        b.synchronize()
        if it >= 5:
            ts.append(a.elapsed_time(b))
    ms = sum(ts) / len(ts)
    print(f"N={world}: rank-0 share {cands} candidates, {ms:.3f} ms/step -> projected whole-job "
          f"{cands * world / ms / 1e6:.2f} x 10^9 candidates/s")
    for e in engines:
        e.close()
