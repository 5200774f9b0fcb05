"""The HTTP search service on the device engine.

Mirrors the reference's search endpoints (/root/reference/pkg/src/llmconf/
service.py:136-236): configured once from a mapping or YAML file naming the
latency databases and extra model files, everything loaded eagerly so bad
paths fail at boot.  The difference is residency: at boot every database is
flattened and uploaded to the GPU once (``Engine.db_handle``), and the
per-(db, model, space) plan templates are cached across requests, so a request
costs one K0 count (the 10^4 cap check, service.py:177-180) plus one device
search.  The reference keeps its CPU memo warm for the same reason
(service.py:1-11).

Error contract (service.py:1-11, 169-180, 226-236): 400 malformed request
with the offending field, 404 unknown database or model name, 413 candidate
space too large, 422 no configuration meets the objectives (with diagnostics
and counts), 200 with the report's JSON bytes -- the same bytes as the CLI's
``search`` output, written from device columns (``run_search_json``).

``SearchService`` holds the logic without a web framework; ``create_app``
wraps it in FastAPI with the reference's routes.  The launch-plan generator
(``/api/v1/generate``, ``generator.py``) and static UI hosting are outside the
hot path and not provided.
"""

from __future__ import annotations

from dataclasses import fields
from pathlib import Path
from typing import Any, Mapping

from . import _native as N
from .database import load_db
from .engine import count_candidates, get_engine, search_json_columns
from .report import REPORT_VERSION
from .specs import (
    BACKENDS,
    SERVING_MODES,
    CandidateSpace,
    ModelConfigError,
    ModelSpec,
    ParallelConfigError,
    WorkloadError,
    SearchError,
    WorkloadSpec,
    load_model_spec,
)

_DATA_DIR = Path(__file__).resolve().parent / "data"


def bundled_models() -> dict[str, ModelSpec]:
    """The reference's bundled desk-scale models, registered before configured ones
    (service.py:87-92, 143): qwen-small and moe-small."""
    out = {}
    for p in sorted((_DATA_DIR / "models").glob("*.json")):
        spec = load_model_spec(p)
        out[spec.name] = spec
    return out


def check_device_limits(model: ModelSpec, workload: WorkloadSpec, space: CandidateSpace) -> None:
    """The device path's size limits as 400s on the offending field.

    The reference has no such limits; requests beyond them are rejected up front
    rather than failing inside the engine with a 500."""
    if not 0 <= space.prefill_pool_cap <= 64 or not 0 <= space.decode_pool_cap <= 64:
        raise ApiError(400, "pool caps must be in [0, 64] on the device engine", field="space")
    if "disaggregated" in workload.modes and space.prefill_pool_cap * space.decode_pool_cap > 256:
        raise ApiError(400, "prefill_pool_cap * decode_pool_cap above 256 is not supported on the device engine",
                       field="space")
    if len(set(workload.gpu_budgets)) > N.LC_MAX_BUDGETS:
        raise ApiError(400, f"at most {N.LC_MAX_BUDGETS} distinct gpu_budgets are supported on the device engine",
                       field="workload")
    if model.moe is not None and model.moe.num_experts > 1024:
        raise ApiError(400, "at most 1024 experts are supported on the device engine", field="model")

MAX_CANDIDATES = 10_000  # service.py:34
MAX_JOBS = 16            # service.py:35
_CONFIG_KEYS = {"databases", "models", "static_dir", "cors_origins"}
_REQUEST_KEYS = {"db", "model", "workload", "space", "jobs"}


class ApiError(Exception):
    """An HTTP status with a field-scoped detail document (service.py:39-50)."""

    def __init__(self, status: int, message: str, field: str | None = None,
                 extra: Mapping[str, Any] | None = None) -> None:
        super().__init__(message)
        self.status = status
        self.detail: dict[str, Any] = {"error": message}
        if field:
            self.detail["field"] = field
        if extra:
            self.detail.update(extra)


def load_config(path: str | Path) -> dict:
    """service.py:73-82."""
    import yaml

    with open(path, encoding="utf-8") as f:
        doc = yaml.safe_load(f) or {}
    if not isinstance(doc, dict):
        raise ValueError(f"{path}: service config must be a mapping")
    unknown = set(doc) - _CONFIG_KEYS
    if unknown:
        raise ValueError(f"{path}: unknown config keys {sorted(unknown)}")
    return doc


def _workload_from_doc(doc) -> WorkloadSpec:
    try:
        if not isinstance(doc, dict):
            raise TypeError("workload must be an object")
        return WorkloadSpec.from_doc(doc)
    except (WorkloadError, TypeError, ValueError) as e:
        raise ApiError(400, str(e), field="workload")


def _model_from_request(value, models: Mapping[str, ModelSpec]) -> ModelSpec:
    """A server-loaded model by name, or an inline specification (service.py:95-107)."""
    if isinstance(value, str):
        model = models.get(value)
        if model is None:
            raise ApiError(404, f"unknown model {value!r}", field="model", extra={"available": sorted(models)})
        return model
    try:
        if not isinstance(value, dict):
            raise TypeError("model must be a name or an object")
        return ModelSpec.from_doc(value)
    except (ModelConfigError, TypeError, ValueError) as e:
        raise ApiError(400, str(e), field="model")


def _space_from_doc(doc) -> CandidateSpace:
    """service.py:110-125."""
    if doc is None:
        return CandidateSpace()
    if not isinstance(doc, dict):
        raise ApiError(400, "space must be an object", field="space")
    known = {f.name for f in fields(CandidateSpace)}
    unknown = sorted(set(doc) - known)
    if unknown:
        raise ApiError(400, f"unknown space fields: {unknown}", field=f"space.{unknown[0]}")
    kwargs = {key: tuple(value) if isinstance(value, list) else value for key, value in doc.items()}
    try:
        return CandidateSpace(**kwargs)
    except (TypeError, ValueError, ParallelConfigError) as e:
        raise ApiError(400, str(e), field="space")


class SearchService:
    """Device-resident search service state: databases, models and the engine."""

    def __init__(self, config: str | Path | Mapping | None = None, bundled: Mapping | None = None,
                 max_candidates: int = MAX_CANDIDATES, device: int = 0, soa_cache: bool = False,
                 upload: bool = True):
        if config is None:
            config = {}
        elif not isinstance(config, Mapping):
            config = load_config(config)
        self.config = dict(config)
        self.databases = {name: load_db(path, soa_cache=soa_cache)
                          for name, path in sorted((config.get("databases") or {}).items())}
        self.models: dict[str, ModelSpec] = bundled_models() if bundled is None else dict(bundled)
        for name, path in sorted((config.get("models") or {}).items()):
            self.models[name] = load_model_spec(path)
        self.max_candidates = max_candidates
        self.device = device
        if upload:
            eng = get_engine(device)
            with eng._lock:
                for db in self.databases.values():
                    eng.db_handle(db)  # flatten + upload once; resident for the process lifetime

    # ---------------------------------------------------------------- endpoints
    def meta(self) -> dict:
        """GET /api/v1/meta (service.py:183-224), without the generator's backend profiles."""
        hardware = {db.hardware.name: db.hardware for db in self.databases.values()}
        return {
            "version": REPORT_VERSION,
            "modes": list(SERVING_MODES),
            "backends": list(BACKENDS),
            "databases": [{"name": name, "backend": db.backend, "backend_version": db.backend_version,
                           "hardware": db.hardware.name, "records": len(db.records)}
                          for name, db in sorted(self.databases.items())],
            "models": [{"name": s.name, "num_layers": s.num_layers, "hidden_size": s.hidden_size,
                        "moe": s.moe is not None, "weight_quant": s.weight_quant}
                       for s in sorted(self.models.values(), key=lambda s: s.name)],
            "hardware": [{"name": h.name, "gpu_memory": h.gpu_memory, "mem_bandwidth": h.mem_bandwidth,
                          "gpus_per_node": h.gpus_per_node}
                         for h in sorted(hardware.values(), key=lambda h: h.name)],
        }

    def validate(self, body) -> dict:
        """The request model's checks (service.py:53-61): extra fields forbidden, jobs in [1, 16]."""
        if not isinstance(body, dict):
            raise ApiError(400, "request body must be an object", field="body")
        extra = sorted(set(body) - _REQUEST_KEYS)
        if extra:
            raise ApiError(400, "Extra inputs are not permitted", field=extra[0])
        for key in ("db", "model", "workload"):
            if key not in body:
                raise ApiError(400, "Field required", field=key)
        if not isinstance(body["db"], str):
            raise ApiError(400, "Input should be a valid string", field="db")
        jobs = body.get("jobs", 1)
        if isinstance(jobs, bool) or not isinstance(jobs, int):
            raise ApiError(400, "Input should be a valid integer", field="jobs")
        if not 1 <= jobs <= MAX_JOBS:
            raise ApiError(400, f"Input should be between 1 and {MAX_JOBS}", field="jobs")
        return body

    def resolve(self, body: dict):
        """service.py:169-180: names -> objects, then the candidate cap (K0 on the device)."""
        db = self.databases.get(body["db"])
        if db is None:
            raise ApiError(404, f"unknown database {body['db']!r}", field="db",
                           extra={"available": sorted(self.databases)})
        model = _model_from_request(body["model"], self.models)
        workload = _workload_from_doc(body["workload"])
        space = _space_from_doc(body.get("space"))
        check_device_limits(model, workload, space)
        try:
            n = count_candidates(model, space, workload, db, device=self.device)
        except (N.EngineLimitError, SearchError) as e:
            raise ApiError(400, str(e), field="space")
        if n > self.max_candidates:
            raise ApiError(413, f"{n} candidates exceed the {self.max_candidates} limit", field="space")
        return db, model, workload, space

    def search(self, body) -> str:
        """POST /api/v1/search (service.py:226-236): the report JSON, or ApiError."""
        body = self.validate(body)
        db, model, workload, space = self.resolve(body)
        try:
            text, cols = search_json_columns(db, model, workload, space, jobs=body.get("jobs", 1),
                                             device=self.device)
        except (N.EngineLimitError, SearchError) as e:
            raise ApiError(400, str(e), field="space")
        if cols.best < 0:
            import json

            doc = json.loads(text)
            raise ApiError(422, "no configuration meets the objectives",
                           extra={"diagnostics": doc["diagnostics"], "counts": doc["counts"]})
        return text


def create_app(config: str | Path | Mapping | None = None, **kwargs):
    """FastAPI application with the reference's search routes (service.py:136-236).

    The search route is a plain function, so FastAPI runs the device call in its
    worker thread pool instead of on the event loop.
    """
    from fastapi import Body, FastAPI, Request, Response
    from fastapi.exceptions import RequestValidationError
    from fastapi.middleware.cors import CORSMiddleware
    from fastapi.responses import JSONResponse

    svc = SearchService(config, **kwargs)
    app = FastAPI(title="llmconf-b200", version=REPORT_VERSION)
    app.state.service = svc
    app.add_middleware(CORSMiddleware, allow_origins=list(svc.config.get("cors_origins") or ["*"]),
                       allow_methods=["*"], allow_headers=["*"])

    @app.exception_handler(ApiError)
    async def on_api_error(request: Request, exc: ApiError) -> JSONResponse:
        return JSONResponse(status_code=exc.status, content={"detail": exc.detail})

    @app.exception_handler(RequestValidationError)
    async def on_validation_error(request: Request, exc: RequestValidationError) -> JSONResponse:
        first = exc.errors()[0]
        field = ".".join(str(part) for part in first["loc"] if part != "body")
        return JSONResponse(status_code=400, content={"detail": {"error": first["msg"], "field": field or "body"}})

    @app.get("/api/v1/meta")
    def meta() -> dict:
        return svc.meta()

    @app.post("/api/v1/search")
    def search(body: Any = Body(...)) -> Response:
        return Response(content=svc.search(body), media_type="application/json")

    return app
