"""The compat layer keeps the reference's public signatures (parameter names, order and
defaults) — pinned by tests/golden/ref_signatures.json, which make_golden.py --signatures
records from the reference package.  CPU only (no device calls)."""

import inspect
import json
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden" / "ref_signatures.json"


def _sig(obj):
    if inspect.isclass(obj):
        obj = obj.__init__
    out = []
    for p in inspect.signature(obj).parameters.values():
        if p.name == "self":
            continue
        out.append([p.name, None if p.default is inspect._empty else repr(p.default)])
    return out


def test_compat_signatures_match_reference():
    from paper_2311_13862_b200 import compat
    ref = json.loads(GOLDEN.read_text())
    for name, params in ref.items():
        obj = getattr(compat, name)
        got = _sig(obj)
        assert [p[0] for p in got] == [p[0] for p in params], name
        assert [p[1] for p in got] == [p[1] for p in params], name


def test_method_registry_matches_reference():
    from paper_2311_13862_b200 import compat
    assert compat.METHODS == ("mgcg", "rbi-mgcg", "rbi-msrbcg")
    cfg = compat.MethodConfig("rbi-mgcg", delta=1e-10, l_max=60, N=4)
    assert (cfg.initializer, cfg.preconditioner) == ("l1roc", "mg")
    assert len(cfg.config_hash()) == 16
