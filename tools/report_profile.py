import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import paper_2601_06288_b200 as pkg
from paper_2601_06288_b200.sweeps import sweep
part = sweep("config5")[0]; w = part.workloads[44]
for _ in range(2): pkg.run_search_json(part.db, part.model, w, part.space)
pr = cProfile.Profile(); pr.enable()
pkg.run_search_json(part.db, part.model, w, part.space)
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
