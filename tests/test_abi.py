"""CPU: the C-ABI library loads, exports every symbol include/*.h declares,
and its host-side contracts (validation, errors) hold. No compute calls."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2001_05291_b200 import _native, fleetplace as F

ROOT = Path(__file__).resolve().parents[1]


def _declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(fp_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    declared = _declared_symbols()
    assert declared, "no declarations found"
    assert declared == set(_native.EXPORTS)
    for name in sorted(declared):
        assert hasattr(lib, name), name


def test_abi_version():
    assert _native.lib().fp_abi_version() == 4


def test_library_is_sm100a_only():
    """The fatbinary carries sm_100a SASS and nothing else (no PTX fallback
    for other architectures, no CPU path)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_device_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    p = C.c_void_p()
    rc = _native.lib().fp_ctx_create(0, C.byref(p))
    assert rc == 8  # FP_ERR_CUDA: no CPU fallback
    with pytest.raises(F.CudaError):
        F.build_distance_table(F.small_generated(1))


def _tiny():
    return F.Instance(
        bases=[(10, 0, (44.0, -79.0)), (11, 0, (46.0, -74.0)), (12, 1, (45.0, -76.0))],
        fleet=[(1, 0), (2, 1)],
        missions=[(100, (45.2, -75.5), (44.8, -76.3), True),
                  (101, (44.2, -78.5), (43.9, -79.2), False)])


def test_validate_instance_contract():
    """proj/src/model.cpp:46-74 (checked on the host, before any kernel)."""
    F.validate_instance(_tiny())
    bad = _tiny()
    bad.base_id[1] = 10
    bad._cstruct = None
    with pytest.raises(F.ValidationError, match="duplicate id"):
        F.validate_instance(bad)
    # duplicate mission ids: the first repeat in load order is reported, for
    # compact id ranges (bitmap) and sparse ones (hash map)
    for ids in ([5, 6, 7, 6, 5], [5, 2_000_000_000, -7, 2_000_000_000, 5]):
        dup = F.Instance(bases=[(1, 0, (45.0, -75.0))], fleet=[(0, 0)],
                         missions=[(i, (45.0, -75.0), (45.5, -75.5), False) for i in ids])
        with pytest.raises(F.ValidationError, match=f"mission {ids[3]}: duplicate id"):
            F.validate_instance(dup)
    ok = F.Instance(bases=[(1, 0, (45.0, -75.0))], fleet=[(0, 0)],
                    missions=[(i, (45.0, -75.0), (45.5, -75.5), False)
                              for i in (2_000_000_000, -2_000_000_000, 0, 3)])
    F.validate_instance(ok)
    bad = _tiny()
    bad.pickup_lat[0] = 91.0
    with pytest.raises(F.ValidationError, match="out of range"):
        F.validate_instance(bad)
    bad = F.Instance(bases=[(1, 1, (45.0, -75.0))], fleet=[(0, 1)], missions=[])
    with pytest.raises(F.ValidationError, match="aerodrome per fixed-wing"):
        F.validate_instance(bad)
    with pytest.raises(F.ValidationError, match="must not be empty"):
        F.validate_instance(F.Instance(bases=[(1, 0, (45.0, -75.0))], fleet=[], missions=[]))


def test_index_views_and_counts():
    inst = _tiny()
    assert inst.base_index(12) == 2 and inst.base_index(99) == -1
    assert inst.vehicle_index(2) == 1 and inst.mission_index(101) == 1
    assert inst.rotary_count() == 1 and inst.fixed_count() == 1
    assert inst.aerodrome_count() == 2 and inst.helipad_count() == 1
    assert [b.id for b in inst.bases] == [10, 11, 12]


def test_check_feasible_rules():
    """proj/src/model.cpp:118-174 restated host-side."""
    inst = _tiny()
    ok = F.Assignment({1: 12, 2: 10}, {100: 1, 101: 2})
    assert F.check_feasible(ok, inst) == []
    bad = F.Assignment({1: 12, 2: 12}, {100: 2, 101: 2})
    rules = {v.rule for v in F.check_feasible(bad, inst)}
    assert rules == {F.Rule.FixedWingOnHelipad, F.Rule.BaseOccupancy, F.Rule.RotaryOnly}
    missing = F.Assignment({1: 12}, {100: 1})
    rules = {v.rule for v in F.check_feasible(missing, inst)}
    assert rules == {F.Rule.OneBasePerVehicle, F.Rule.OneVehiclePerMission}


def test_initial_pool_order():
    """proj/src/search.cpp:364-377: unused bases in ranking order, then idle
    placed vehicles by vehicle id."""
    start = F.RankedStart(F.Assignment({7: 1, 3: 2, 5: 0}, {0: 7}), [4, 3], np.zeros(5))
    pool = F.initial_pool(start, None)
    assert pool == [F.PoolEntry(F.PoolEntryKind.EmptyBase, 4), F.PoolEntry(F.PoolEntryKind.EmptyBase, 3),
                    F.PoolEntry(F.PoolEntryKind.IdleVehicle, 3), F.PoolEntry(F.PoolEntryKind.IdleVehicle, 5)]


def test_struct_field_views_match_ctypes():
    """fleetplace._fields (the vectorised marshalling of search_batch) views
    exactly the bytes ctypes reads and writes, nested stats included."""
    import ctypes as C
    import numpy as np
    from paper_2001_05291_b200 import _abi as A
    from paper_2001_05291_b200 import fleetplace as F
    n = 5
    res = (A.fp_search_result * n)()
    for k in range(n):
        res[k].stats.evaluations = 1000 + k
        res[k].stats.final_objective_km = 0.5 * k
        res[k].device_ms = 2.0 * k
        res[k].kernel_launches = 7 * k
    rv = F._fields(res, A.fp_search_result, n)
    ss = F._fields(res, A.fp_search_result, n, nested="stats")
    assert ss["evaluations"].tolist() == [1000 + k for k in range(n)]
    assert ss["final_objective_km"].tolist() == [0.5 * k for k in range(n)]
    assert rv["device_ms"].tolist() == [2.0 * k for k in range(n)]
    assert rv["kernel_launches"].tolist() == [7 * k for k in range(n)]
    buf = np.arange(10, dtype=np.int32)
    rv["mission_vehicle"][:] = buf.ctypes.data + 4 * np.arange(n)
    for k in range(n):
        assert C.cast(res[k].mission_vehicle, C.c_void_p).value == buf.ctypes.data + 4 * k
        assert res[k].mission_vehicle[0] == k
    st = (A.fp_search_start * n)()
    sv = F._fields(st, A.fp_search_start, n)
    sv["pool_size"][:] = np.arange(n) + 3
    assert [st[k].pool_size for k in range(n)] == [3 + k for k in range(n)]


def test_bench_parity_gate_and_goldens():
    """bench.py's parity gate accepts the reference's recorded c2 run and
    refuses a trajectory that differs in any counter or in the Assignment."""
    import importlib.util
    import types
    from pathlib import Path

    import numpy as np
    import pytest as _pt
    spec = importlib.util.spec_from_file_location("bench_mod", Path(__file__).resolve().parents[1] / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    g = bench._golden("c2_full")
    st = types.SimpleNamespace(passes=g["stats"][0], evaluations=g["stats"][1],
                               applied_moves=g["stats"][2], committed_moves=g["stats"][3],
                               tabu_skips_outer=g["stats"][4], tabu_skips_inner=g["stats"][5],
                               final_objective_km=g["final_objective_km"])
    vb = np.array(g["vehicle_base"], np.int32)
    mv = np.array(g["mission_vehicle"], np.int32)
    bench._assert_golden("c2_full", st, vb, mv)  # the reference's own run passes
    bad = types.SimpleNamespace(**{**vars(st), "evaluations": st.evaluations + 1})
    with _pt.raises(SystemExit):
        bench._assert_golden("c2_full", bad, vb, mv)
    mv2 = mv.copy()
    mv2[0] = (mv2[0] + 1) % 40
    with _pt.raises(SystemExit):
        bench._assert_golden("c2_full", st, vb, mv2)
