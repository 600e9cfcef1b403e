"""bench.py's CPU side (the `--impl reference` arm and the `cpu_baseline`
leg): runs without the reference installed (oracle port), never imports the
product package, reports what it measured apart from what it extrapolates,
and builds the reference's own cavity mesh (oracle/fvcases.py)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from golden_io import load as golden_npz
from oracle import fvcases

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name,args", [
    ("cav6", (6, 6, 6, 0.1, 0.1, 0.1, [("lid", "wall", ["y+"]),
                                       ("walls", "wall", ["x-", "x+", "y-", "z-", "z+"])])),
    ("cav20", (20, 20, 1, 0.1, 0.1, 0.01, [("movingWall", "wall", ["y+"]),
                                          ("fixedWalls", "wall", ["x-", "x+", "y-"]),
                                          ("frontAndBack", "empty", ["z-", "z+"])])),
    ("chan", (12, 4, 1, 0.16, 0.02, 0.005, [("inlet", "inlet", ["x-"]),
                                           ("outlet", "outlet", ["x+"]),
                                           ("walls", "wall", ["y-", "y+"]),
                                           ("frontAndBack", "empty", ["z-", "z+"])])),
])
def test_oracle_box_mesh_is_the_reference_mesh(name, args):
    g = golden_npz(name)
    m = fvcases.box_mesh(*args)
    for k in ("points", "face_points", "face_offsets", "owner", "neighbour"):
        assert np.array_equal(getattr(m, k), g[k]), k
    assert [p.name for p in m.patches] == list(g["patch_names"])
    assert [p.start for p in m.patches] == list(g["patch_start"])
    assert [p.count for p in m.patches] == list(g["patch_count"])


def test_reference_arm_runs_without_the_product():
    code = (
        "import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--edge', '10', "
        "'--steps', '2', '--warmup', '1', '--cg-sample', '5']\n"
        "import bench\n"
        "bench.REF_DIR = '/nonexistent'\n"
        "bench.main()\n"
        "assert not any(m.startswith('paper_1207_1571_b200') for m in sys.modules), 'product imported'\n"
    )
    out = subprocess.run([sys.executable, "-c", code], cwd=REPO, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "port"
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    meas = line["measured"]
    assert meas["cells"] == 1000 and meas["samples"] == 2
    assert meas["iters_per_sample"]["cg"] <= 2 * 5
    # the measured sample is what ran: steps x ms_per_step is its wall time
    assert abs(line["ms_per_step"] / 1e3 - meas["s_per_sample"]) < 1e-9
    assert line["extrapolated"]["cell_scale"] == 1.0
    assert line["one_thread"]["value"] > 0
