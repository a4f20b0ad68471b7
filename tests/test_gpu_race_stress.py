"""Dynamic race check of the synchronisation protocols (cluster barriers,
DSMEM st.async + mbarrier, shared-memory transposes, the cooperative grid
sync, the compact plan's cluster agreement): one small invocation of every
kernel family against the race-stress build of the library (-DBW_RACE_STRESS:
random warp sleeps at every synchronisation point), each compared bit for
bit with the CPU oracle.  compute-sanitizer is closed on this GPU pool, so
this replaces racecheck / synccheck (tools/race_stress.sh runs it repeatedly)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STRESS = os.path.join(ROOT, "paper_1607_01039_b200", "lib", "libbigwht_b200_stress.so")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(STRESS), reason="race-stress build missing (build.py --stress)")
def test_every_kernel_family_under_race_stress():
    env = dict(os.environ, BW_LIB_PATH=STRESS)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MISMATCH" not in r.stdout
    assert "done all" in r.stdout
