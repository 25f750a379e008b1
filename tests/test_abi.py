"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol include/pfc.h declares,
and host-detectable configuration errors are returned synchronously (pfc.h conventions)."""
import ctypes
import os
import re

import pytest

import paper_2010_05222_b200 as pfc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pfc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pfc_[a-z_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = pfc.load_library()
    names = _declared()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(names) == sorted(pfc.EXPORTS)
    assert b"sm_100a" in lib.pfc_version()


def _cfg(**kw):
    base = dict(num_classes=1000, dim=128, batch=8, sample_rate=0.1, scale=64.0, margin_type=1, margin=0.5,
                momentum=0.9, weight_decay=0.0, precision=1, seed=0, rank=0, world_size=1, device=0,
                nccl_unique_id=None, comm_mode=0, sample_mode=0, param_location=0)
    base.update(kw)
    return pfc._Config(**base)


@pytest.mark.parametrize("bad", [
    dict(sample_rate=0.0), dict(sample_rate=1.5), dict(num_classes=3, world_size=4, rank=0, comm_mode=1),
    dict(dim=100), dict(batch=0), dict(scale=0.0), dict(margin_type=1, margin=1.6), dict(margin_type=2, margin=1.0),
    dict(margin_type=7), dict(precision=3), dict(rank=2, world_size=2, comm_mode=1), dict(world_size=2, rank=0),
    dict(momentum=1.0), dict(comm_mode=5), dict(sample_mode=3), dict(sample_mode=-1), dict(param_location=2),
    dict(param_location=-1),
])
def test_config_errors_are_reported_synchronously(bad):
    lib = pfc.load_library()
    h = ctypes.c_void_p(123)
    s = lib.pfc_init(ctypes.byref(_cfg(**bad)), ctypes.byref(h))
    assert s == 1, (bad, s)                      # PFC_ERR_CONFIG
    assert h.value is None
    assert len(lib.pfc_last_error(None)) > 0


def test_null_arguments_are_contract_errors():
    lib = pfc.load_library()
    assert lib.pfc_init(None, None) == 2
    assert lib.pfc_step(None, ctypes.c_float(0.1), None) == 2
    assert lib.pfc_forward_backward(None, None, None, None, None, None) == 2
    assert lib.pfc_destroy(None) == 0
