"""GPU: the reference's own acceptance suite (proj/tests/acceptance.cpp) run
twice — against the reference's CPU build (oracle/_ref/acceptance) and with
its five hot-path entry points replaced by the B200 drop-in
(oracle/_ref/acceptance_b200 = reference sources with build_distance_table,
column_totals, rank_bases, local_search, tabu_search compiled out, plus
integration/fleetplace_b200_adapter.cpp over the C ABI). Every deterministic
criterion must print the same line; the exit code (unexpected failures) must
be 0 for both."""
import re
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REF = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


def _run(name):
    exe = REF / name
    if not exe.exists():
        pytest.skip(f"{exe} not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600, cwd=REF)
    lines = {int(m.group(1)): m.group(2) for m in
             (re.match(r"\[\s*(\d+)\] (.*)", l) for l in r.stdout.splitlines()) if m}
    return r.returncode, lines


def test_reference_acceptance_suite_on_the_drop_in():
    rc_cpu, cpu = _run("acceptance")
    rc_gpu, gpu = _run("acceptance_b200")
    assert rc_cpu == 0 and rc_gpu == 0, (rc_cpu, rc_gpu)
    # deterministic criteria: identical text (verdict and numbers)
    for k in (1, 2, 3, 4, 5, 7, 8, 9):
        assert gpu[k] == cpu[k], (k, cpu[k], gpu[k])
    # 6 compares against the nondeterministic parallel_tabu_search: verdict only
    assert gpu[6].startswith("PASS") and cpu[6].startswith("PASS")


def test_adapter_objective_and_feasibility_match_reference():
    """The drop-in's O(M) check_feasible and objective_km (device sum) equal
    the reference's O(M^2) ones on fuzzed and ranked assignments."""
    exe = REF / "adapter_check"
    if not exe.exists():
        pytest.skip(f"{exe} not built")
    r = subprocess.run([str(exe), "--gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout and " 0 objectives" not in r.stdout
