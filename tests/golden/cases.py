"""Named search cases shared by the golden generator and the parity tests.

Each case is plain data so it can be turned into reference ``llmconf`` objects
(``make_golden.py``, run in the survey container where /root/reference exists)
or into this package's objects (tests, on the GPU box).  The four BASELINE
configs come first, then the reference's acceptance A1 search
(/root/reference/pkg/tests/test_acceptance.py:81-90), then edge cases chosen to
hit every branch of the path: extrapolation policies, skip reasons, chunking
regimes, osl 1/2, prefix reuse, flat (tie-heavy) databases, empty fronts.
"""

from __future__ import annotations

W45 = dict(isl=4000, osl=500, ttft_limit_ms=1200.0, min_speed=60.0)

CASES: list[dict] = [
    # --- BASELINE.json configs 1-4 -------------------------------------------------
    dict(name="cfg1_qwen3_agg", model="qwen3-32b",
         workload=dict(W45, gpu_budgets=[8], modes=["aggregated"]), space=dict(pp_values=[1])),
    dict(name="cfg2_qwen3_disagg", model="qwen3-32b",
         workload=dict(W45, gpu_budgets=[8], modes=["disaggregated"]), space=dict(pp_values=[1])),
    *[
        dict(name=f"cfg3_llama70b_kv{int(f * 100)}", model="llama-3.1-70b",
             workload=dict(W45, gpu_budgets=[8, 16], modes=["aggregated", "disaggregated"]),
             space=dict(kv_mem_fraction=f))
        for f in (0.5, 0.7, 0.9)
    ],
    dict(name="cfg4_dsv3", model="deepseek-v3",
         workload=dict(isl=5000, osl=1000, ttft_limit_ms=5000.0, min_speed=20.0, gpu_budgets=[8, 16]),
         space={}),
    # --- acceptance A1 and full default spaces -------------------------------------
    dict(name="a1_qwen_small", model="qwen-small",
         workload=dict(isl=512, osl=64, ttft_limit_ms=10000.0, min_speed=1.0), space={}),
    dict(name="qwen3_all_default", model="qwen3-32b", workload=dict(W45), space={}),
    dict(name="dsv3_all_default", model="deepseek-v3",
         workload=dict(isl=4000, osl=500, ttft_limit_ms=5000.0, min_speed=20.0), space={}),
    dict(name="gptoss_all_default", model="gpt-oss-120b", workload=dict(W45), space={}, large=True),
    dict(name="moe_small_all", model="moe-small",
         workload=dict(isl=1024, osl=128, ttft_limit_ms=2000.0, tpot_limit_ms=50.0), space={}),
    # --- extrapolation policies ----------------------------------------------------
    dict(name="strict_long_isl", model="qwen-small", extrapolation="strict",
         workload=dict(isl=20000, osl=64, ttft_limit_ms=60000.0, min_speed=1.0),
         space=dict(tp_values=[1, 2], pp_values=[1], dp_values=[1], batch_values=[1, 4, 64])),
    dict(name="clamp_long_isl", model="qwen-small", extrapolation="clamp",
         workload=dict(isl=20000, osl=300, ttft_limit_ms=60000.0, min_speed=1.0),
         space=dict(tp_values=[1, 2], pp_values=[1, 2], dp_values=[1], batch_values=[1, 4, 64, 2048])),
    dict(name="sol_long_isl", model="qwen-small", extrapolation="sol",
         workload=dict(isl=20000, osl=300, ttft_limit_ms=60000.0, min_speed=1.0),
         space=dict(tp_values=[1, 2], pp_values=[1, 2], dp_values=[1], batch_values=[1, 4, 64, 2048])),
    dict(name="default_big_batch", model="moe-small",
         workload=dict(isl=3000, osl=40, ttft_limit_ms=60000.0, min_speed=1.0),
         space=dict(batch_values=[1, 3, 100, 1500, 4096], dp_values=[1, 8])),
    # --- skip reasons ----------------------------------------------------------------
    dict(name="unsupported_quant_a100", model="qwen-small", mutation="swap_hw:a100-sxm",
         workload=dict(isl=20000, osl=64, ttft_limit_ms=60000.0, min_speed=1.0),
         space=dict(tp_values=[1, 2], pp_values=[1], dp_values=[1], batch_values=[1, 8])),
    dict(name="missing_allreduce", model="qwen-small", mutation="drop_kind:allreduce",
         workload=dict(isl=512, osl=64, ttft_limit_ms=10000.0, min_speed=1.0),
         space=dict(tp_values=[1, 2, 4], pp_values=[1, 2], dp_values=[1], batch_values=[1, 16])),
    dict(name="missing_tp16", model="moe-small",
         workload=dict(isl=512, osl=64, ttft_limit_ms=10000.0, min_speed=1.0),
         space=dict(tp_values=[1, 16], pp_values=[1], ep_values=[1, 2], dp_values=[1, 2],
                    batch_values=[2, 32])),
    dict(name="no_chunking", model="qwen-small",
         workload=dict(isl=3000, osl=64, ttft_limit_ms=10000.0, min_speed=1.0),
         space=dict(ctx_capacity=2048, chunked_prefill=False, pp_values=[1], dp_values=[1])),
    dict(name="small_ctx_capacity", model="qwen-small",
         workload=dict(isl=3000, osl=64, ttft_limit_ms=10000.0, min_speed=1.0),
         space=dict(ctx_capacity=512, pp_values=[1, 2], dp_values=[1])),
    dict(name="batch_too_small", model="qwen-small",
         workload=dict(isl=512, osl=200, ttft_limit_ms=10000.0, min_speed=1.0),
         space=dict(ctx_capacity=4096, pp_values=[1], dp_values=[1], batch_values=[1, 2, 4, 8, 9, 16, 64])),
    # --- workload shapes --------------------------------------------------------------
    dict(name="osl1", model="qwen-small", workload=dict(isl=512, osl=1, ttft_limit_ms=10000.0),
         space=dict(pp_values=[1, 2], dp_values=[1, 2])),
    dict(name="osl2", model="moe-small", workload=dict(isl=700, osl=2, min_speed=1.0),
         space=dict(pp_values=[1, 2], dp_values=[1, 2])),
    dict(name="prefix_reuse", model="qwen-small",
         workload=dict(isl=4096, osl=100, prefix_len=3000, ttft_limit_ms=10000.0, min_speed=5.0),
         space=dict(pp_values=[1, 4])),
    dict(name="batch_sweep_override", model="moe-small",
         workload=dict(isl=900, osl=77, batch_sweep=[3, 1, 48, 7], ttft_limit_ms=8000.0, min_speed=2.0),
         space={}),
    dict(name="no_sla", model="qwen-small", workload=dict(isl=256, osl=32),
         space=dict(pp_values=[1], dp_values=[1, 2])),
    dict(name="unmeetable_sla", model="qwen-small",
         workload=dict(isl=512, osl=32, ttft_limit_ms=5000.0, min_speed=1e9),
         space=dict(tp_values=[1, 2], pp_values=[1], dp_values=[1], batch_values=[1, 8, 64])),
    dict(name="unmeetable_ttft", model="moe-small",
         workload=dict(isl=2048, osl=32, ttft_limit_ms=0.001, min_speed=1.0),
         space=dict(pp_values=[1], dp_values=[1, 2])),
    dict(name="disagg_constants", model="qwen-small",
         workload=dict(isl=2048, osl=256, ttft_limit_ms=3000.0, min_speed=10.0, gpu_budgets=[4, 8, 12]),
         space=dict(prefill_pool_cap=3, decode_pool_cap=5),
         disagg=dict(ttft_headroom=1.5, prefill_utilization=0.8, decode_utilization=0.95,
                     max_prefill_replicas=5, max_decode_replicas=7)),
    dict(name="moe_load_custom", model="moe-small",
         workload=dict(isl=1500, osl=90, ttft_limit_ms=5000.0, min_speed=5.0,
                       moe_load=dict(alpha=0.5, x_min=1.0, x_max=1000.0, seed=3)),
         space=dict(dp_values=[1, 2, 8])),
    dict(name="moe_load_uniform", model="moe-small",
         workload=dict(isl=700, osl=50, min_speed=3.0, moe_load=dict(alpha=0.0, x_min=1.0, x_max=2.0, seed=9)),
         space=dict(pp_values=[1], dp_values=[2, 4])),
    dict(name="flat_ties", model="qwen-small", mutation="flat",
         workload=dict(isl=512, osl=33, ttft_limit_ms=10000.0, min_speed=1.0), space={}),
    dict(name="flat_ties_moe", model="moe-small", mutation="flat",
         workload=dict(isl=600, osl=65, min_speed=0.5), space=dict(pp_values=[1, 2])),
    dict(name="dsv3_b200_pp1", model="deepseek-v3", hw="b200-sxm",
         workload=dict(isl=5000, osl=1000, ttft_limit_ms=5000.0, min_speed=20.0, gpu_budgets=[8, 16]),
         space=dict(pp_values=[1])),
]

BY_NAME = {c["name"]: c for c in CASES}

# databases: one synthetic DB per (model, hardware), reference dbgen with seed 11
# (/root/reference/pkg/src/llmconf/perfdb.py:641-666, model.py:509-545)
DB_SEED = 11


def db_file(model: str, hw: str = "h100-sxm") -> str:
    return f"db-{model}-{hw}-s{DB_SEED}.jsonl.gz"


def case_db_key(case: dict) -> tuple[str, str]:
    return case["model"], case.get("hw", "h100-sxm")
