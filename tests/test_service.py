"""Search service: the reference's error contract
(/root/reference/pkg/tests/test_service.py:86-150) on this package's service.

CPU tests cover everything decided before the device is touched (meta, 400,
404); the -m gpu tests cover 200 (report bytes equal the reference's golden
report), 413 (K0 count over the cap), 422 (diagnostics) and residency (each
database uploaded once, at boot)."""

from __future__ import annotations

import json

import pytest

from golden_io import BY_NAME, db_path, golden_report

ROOT_SPECS = __import__("pathlib").Path(__file__).resolve().parent / "golden" / "specs"


def _config():
    case = BY_NAME["a1_qwen_small"]
    return {"databases": {"qwen-h100": str(db_path(case)),
                          "dsv3-h100": str(db_path(BY_NAME["cfg4_dsv3"]))},
            "models": {n: str(ROOT_SPECS / f"model-{n}.json") for n in ("qwen-small", "moe-small", "deepseek-v3")}}


def _body(**over):
    case = BY_NAME["a1_qwen_small"]
    body = {"db": "qwen-h100", "model": "qwen-small", "workload": dict(case["workload"]), "space": {}}
    body.update(over)
    return body


@pytest.fixture(scope="module")
def cpu_client():
    from fastapi.testclient import TestClient

    from paper_2601_06288_b200.service import create_app

    return TestClient(create_app(_config(), upload=False))


def test_meta_lists_databases_models_hardware(cpu_client):
    doc = cpu_client.get("/api/v1/meta").json()
    assert [d["name"] for d in doc["databases"]] == ["dsv3-h100", "qwen-h100"]
    assert [m["name"] for m in doc["models"]] == ["deepseek-v3", "moe-small", "qwen-small"]
    assert doc["modes"] == ["static", "aggregated", "disaggregated"]
    assert [h["name"] for h in doc["hardware"]] == ["h100-sxm"]
    assert doc == cpu_client.get("/api/v1/meta").json()


def test_unknown_database_404_names_field(cpu_client):
    resp = cpu_client.post("/api/v1/search", json=_body(db="nope"))
    assert resp.status_code == 404
    assert resp.json()["detail"] == {"error": "unknown database 'nope'", "field": "db",
                                     "available": ["dsv3-h100", "qwen-h100"]}


def test_unknown_model_404(cpu_client):
    resp = cpu_client.post("/api/v1/search", json=_body(model="nope"))
    assert resp.status_code == 404
    assert resp.json()["detail"]["field"] == "model"


def test_bad_inline_model_400(cpu_client):
    resp = cpu_client.post("/api/v1/search", json=_body(model={"name": "x"}))
    assert resp.status_code == 400
    assert resp.json()["detail"]["field"] == "model"


def test_malformed_jobs_400_with_field(cpu_client):
    for jobs in ("many", 0, 17):
        resp = cpu_client.post("/api/v1/search", json=_body(jobs=jobs))
        assert resp.status_code == 400
        assert resp.json()["detail"]["field"] == "jobs"


def test_bad_workload_field_400(cpu_client):
    body = _body()
    body["workload"]["surprise"] = 1
    resp = cpu_client.post("/api/v1/search", json=body)
    assert resp.status_code == 400
    detail = resp.json()["detail"]
    assert detail["field"] == "workload" and "surprise" in detail["error"]


def test_unknown_space_field_400(cpu_client):
    resp = cpu_client.post("/api/v1/search", json=_body(space={"warp": 9}))
    assert resp.status_code == 400
    assert resp.json()["detail"]["field"] == "space.warp"


def test_extra_request_field_400(cpu_client):
    resp = cpu_client.post("/api/v1/search", json=_body(surprise=1))
    assert resp.status_code == 400
    assert resp.json()["detail"]["field"] == "surprise"


def test_bundled_models_registered_without_config():
    """create_app registers the reference's bundled models (service.py:87-92, 143)."""
    from fastapi.testclient import TestClient

    from paper_2601_06288_b200.service import create_app

    client = TestClient(create_app({"databases": {"qwen-h100": str(db_path(BY_NAME["a1_qwen_small"]))}},
                                   upload=False))
    assert [m["name"] for m in client.get("/api/v1/meta").json()["models"]] == ["moe-small", "qwen-small"]
    for name in ("qwen-small", "moe-small"):
        assert json.loads((ROOT_SPECS / f"model-{name}.json").read_text()) == json.loads(
            (ROOT_SPECS.parents[2] / "paper_2601_06288_b200" / "data" / "models" / f"{name}.json").read_text())


@pytest.mark.parametrize("space,workload_over,field", [
    ({"prefill_pool_cap": 65}, {}, "space"),
    ({"prefill_pool_cap": 32, "decode_pool_cap": 16}, {}, "space"),
    ({}, {"gpu_budgets": list(range(1, 18))}, "workload"),
])
def test_device_limits_are_400(cpu_client, space, workload_over, field):
    body = _body(space=space)
    body["workload"] = dict(body["workload"], **workload_over)
    resp = cpu_client.post("/api/v1/search", json=body)
    assert resp.status_code == 400
    assert resp.json()["detail"]["field"] == field


def test_config_file_rejects_unknown_keys(tmp_path):
    from paper_2601_06288_b200.service import load_config

    p = tmp_path / "svc.yaml"
    p.write_text("databases: {}\nsurprise: 1\n")
    with pytest.raises(ValueError, match="unknown config keys"):
        load_config(p)


# ------------------------------------------------------------------ on the GPU
@pytest.fixture(scope="module")
def gpu_client():
    from fastapi.testclient import TestClient

    from paper_2601_06288_b200.service import create_app

    return TestClient(create_app(_config()))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["a1_qwen_small", "cfg4_dsv3"])
def test_search_returns_reference_report_bytes(gpu_client, name):
    case = BY_NAME[name]
    db = "qwen-h100" if case["model"] == "qwen-small" else "dsv3-h100"
    body = {"db": db, "model": case["model"], "workload": dict(case["workload"]), "space": dict(case["space"])}
    resp = gpu_client.post("/api/v1/search", json=body)
    assert resp.status_code == 200
    doc = json.loads(resp.content)
    doc.pop("timing")
    golden = golden_report(name)
    golden.pop("_meta")
    assert json.dumps(doc, sort_keys=True) == json.dumps(golden, sort_keys=True)
    again = json.loads(gpu_client.post("/api/v1/search", json=dict(body, jobs=4)).content)
    again.pop("timing")
    assert again == doc


@pytest.mark.gpu
def test_no_feasible_configuration_422_with_diagnostics(gpu_client):
    body = _body()
    body["workload"]["min_speed"] = 1e9
    resp = gpu_client.post("/api/v1/search", json=body)
    assert resp.status_code == 422
    detail = resp.json()["detail"]
    assert detail["diagnostics"]["violation_factor"] > 1
    assert detail["counts"]["feasible"] == 0


@pytest.mark.gpu
def test_oversized_candidate_space_413(gpu_client):
    body = _body(workload={"isl": 64, "osl": 16},
                 space={"batch_values": list(range(1, 1501)), "tp_values": [1, 2], "pp_values": [1, 2, 4],
                        "dp_values": [1, 2]})
    resp = gpu_client.post("/api/v1/search", json=body)
    assert resp.status_code == 413
    assert "candidates" in resp.json()["detail"]["error"]


@pytest.mark.gpu
def test_databases_resident_after_boot(gpu_client):
    from paper_2601_06288_b200.engine import get_engine

    svc = gpu_client.app.state.service
    eng = get_engine(0)
    handles = {name: eng._dbs[id(db)][0].value for name, db in svc.databases.items()}
    gpu_client.post("/api/v1/search", json=_body())
    assert {name: eng._dbs[id(db)][0].value for name, db in svc.databases.items()} == handles
