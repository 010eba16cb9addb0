"""The C-ABI library loads and exports every symbol include/*.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

import paper_2011_01112_b200 as pkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"^\s*(?:int|int64_t)\s+(ic_\w+)\s*\(", txt, flags=re.M))


def test_library_exports_every_declared_symbol():
    lib = pkg.load_library()
    declared = (_declared("ic_sched.h") | _declared("ic_sim.h") | _declared("ic_probe.h")
                | (_declared("ic_gen.h") - {"ic_gen_batch_host"}))
    assert declared == set(pkg.abi.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name


def test_host_generator_symbol():
    import gen
    lib = gen._load()
    assert hasattr(lib, "ic_gen_batch_host")


def test_invalid_configs_rejected_before_cuda():
    lib = pkg.load_library()
    h = ctypes.c_void_p()
    bad = [pkg.SchedConfig(delta_micro=0, epsilon_micro=0),
           pkg.SchedConfig(drop_mode=7),
           pkg.SchedConfig(max_tasks=0)]
    for c in bad:
        assert lib.ic_sched_create(ctypes.byref(c), ctypes.byref(h)) == pkg.IC_ERR_INVALID_ARG
    for c in (pkg.SchedConfig(max_tasks=5000), pkg.SchedConfig(max_opt_stages=15),
              pkg.SchedConfig(max_horizon=40000)):
        assert lib.ic_sched_create(ctypes.byref(c), ctypes.byref(h)) == pkg.IC_ERR_LIMIT
    assert lib.ic_sched_create(None, ctypes.byref(h)) == pkg.IC_ERR_INVALID_ARG
    assert lib.ic_sched_solve_batch(None, None, None, None) == pkg.IC_ERR_INVALID_ARG
    assert lib.ic_sched_destroy(None) == pkg.IC_ERR_INVALID_ARG


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(pkg.ICSchedError) as e:
        pkg.Scheduler(pkg.SchedConfig())
    assert e.value.rc == pkg.IC_ERR_CUDA


def test_product_package_does_not_import_oracle():
    """The product path must never route through oracle/ (task brief ③)."""
    pdir = os.path.join(ROOT, "paper_2011_01112_b200")
    for dirpath, _, files in os.walk(pdir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                for pat in ("import oracle", "from oracle", "liboracle", "ic_oracle"):
                    assert pat not in src, (f, pat)


def test_to_micro_quantises_like_the_spec():
    """The wrapper's float -> micro-unit conversion (SURVEY §8(b) "Wrapper", D5/G11): the
    decimal examples of S:L180-182 and S:L190 quantise as the spec says once the confidences
    are micro-units (fp64 floor(0.7/0.1) would give 6), and ties round half to even."""
    import torch
    from paper_2011_01112_b200 import to_micro, confidences_to_inputs
    delta = 100_000  # Delta = 0.1
    q = to_micro([0.57, 1.0, 0.09, 0.7, 0.3, 0.6], torch.int64) // delta
    assert q.tolist() == [5, 10, 0, 7, 3, 6]
    assert to_micro([0.5e-6, 1.5e-6, 2.5e-6, 3.5e-6]).tolist() == [0, 2, 2, 4]
    m, g = confidences_to_inputs(torch.tensor([0.3, 0.5], dtype=torch.float64),
                                 torch.tensor([[0.4, 0.7], [0.55, 0.6]], dtype=torch.float64))
    assert m.dtype == torch.uint32 and g.dtype == torch.int32
    assert m.to(torch.int64).tolist() == [300000, 500000]
    assert g.tolist() == [[100000, 300000], [50000, 50000]]
    with pytest.raises(ValueError):
        to_micro([float("nan")])
    with pytest.raises(ValueError):
        to_micro([-0.1], torch.uint32)


def _struct_fields(header, name):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    end = re.search(r"\}\s*" + name + ";", txt).start()
    body = txt[txt.rindex("typedef struct {", 0, end) + len("typedef struct {"):end]
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        m = re.match(r"(u?int(?:32|64)_t)\s+(.*)", decl)
        assert m, decl
        fields += [(m.group(1), f.strip()) for f in m.group(2).split(",")]
    return fields


def test_tuning_and_info_structs_match_the_header():
    """The binding's ctypes mirrors of ic_sched_tuning and ic_sched_info have the header's fields
    in the header's order and widths (both grew this round: packed_options, discard)."""
    import ctypes
    tun = _struct_fields("ic_sched.h", "ic_sched_tuning")
    assert [n for _, n in tun] == list(pkg.TUNING_FIELDS)
    assert all(t == "int32_t" for t, _ in tun)
    info = _struct_fields("ic_sched.h", "ic_sched_info")
    got = [(n, ctypes.sizeof(t)) for n, t in pkg.SchedInfo._fields_]
    assert got == [(n, 8 if t.endswith("64_t") else 4) for t, n in info]
