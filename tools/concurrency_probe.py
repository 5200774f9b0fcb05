import sys
sys.path.insert(0, '.')
import torch
from paper_2601_06288_b200.engine import Engine
from paper_2601_06288_b200.sweeps import sweep
parts = sweep("config5")
def run(copies):
    engines = []
    for c in range(copies):
        for p in parts:
            e = Engine(0); e.run_batch(p.db, p.model, p.space, p.workloads); engines.append(e)
    streams = [torch.cuda.ExternalStream(e.stream_ptr()) for e in engines]
    cur = torch.cuda.current_stream(); ts = []
    for it in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        for st in streams: st.wait_event(a)
        for e in engines: e.replay_async()
        for st in streams:
            d = torch.cuda.Event(); d.record(st); cur.wait_event(d)
        b.record(cur); b.synchronize()
        if it >= 5: ts.append(a.elapsed_time(b))
    print(copies, "copies:", sum(ts)/len(ts), "ms")
    for e in engines: e.close()
run(1); run(2); run(3)
