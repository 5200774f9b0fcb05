"""Diagnose step-latency mismatches against tests/golden/steps.json.gz (prints per-label diffs)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import test_gpu_steps as T  # noqa: E402

bad = 0
for key, recs in sorted(T._groups().items(), key=lambda kv: str(kv[0])):
    got = T._run(key, recs)
    nb = 0
    for r, g in zip(recs, got):
        try:
            T._assert_same(r, g)
        except AssertionError:
            nb += 1
            if nb <= 2:
                print(key, r["cfg"], r["phase"], r["n_ctx"], r["n_gen"], r["seq"], r["moe_load"], r.get("error"))
                if isinstance(g, Exception):
                    print("   got exception", type(g).__name__, g)
                elif "breakdown" in r:
                    gb = {k: v.hex() for k, v in g.breakdown.items()}
                    for k, v in r["breakdown"]:
                        print(f"   {k:24s} ref {v:26s} got {gb.get(k)}", "" if gb.get(k) == v else "  <<<")
                    print("   extra labels:", [k for k in gb if k not in dict(r["breakdown"])])
                else:
                    print("   got", g)
    print(key, "mismatches", nb, "of", len(recs))
    bad += nb
print("total mismatches", bad)
