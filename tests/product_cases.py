"""Build this package's objects for a golden case (no reference import)."""

from __future__ import annotations

import paper_2601_06288_b200 as pkg
from paper_2601_06288_b200.database import with_records
from paper_2601_06288_b200.database import OperatorRecord

from golden_io import db_path, hw_doc, model_doc

_DB_CACHE: dict = {}


def case_db(case: dict):
    key = (str(db_path(case)), case.get("extrapolation", "default"), case.get("mutation"))
    if key in _DB_CACHE:
        return _DB_CACHE[key]
    db = pkg.load_db(db_path(case), extrapolation=case.get("extrapolation", "default"))
    mut = case.get("mutation")
    if mut == "flat":
        db = with_records(db, [OperatorRecord(r.kind, r.quant, r.shape, 100.0, "synthetic") for r in db.records])
    elif mut and mut.startswith("swap_hw:"):
        db = with_records(db, hardware=pkg.HardwareSpec.from_doc(hw_doc(mut.split(":", 1)[1])))
    elif mut and mut.startswith("drop_kind:"):
        kind = mut.split(":", 1)[1]
        db = with_records(db, [r for r in db.records if r.kind != kind])
    _DB_CACHE[key] = db
    return db


def case_objects(case: dict):
    model = pkg.ModelSpec.from_doc(model_doc(case["model"]))
    workload = pkg.WorkloadSpec.from_doc(dict(case["workload"]))
    sp = {k: tuple(v) if isinstance(v, list) else v for k, v in case.get("space", {}).items()}
    space = pkg.CandidateSpace(**sp)
    dc = pkg.DisaggConstants(**case["disagg"]) if case.get("disagg") else pkg.DEFAULT_DISAGG
    return case_db(case), model, workload, space, dc
