"""Host-side tools: the equal-resolution comparison (tools/tgv_compare.py) and the bench workload
names (bench.make_case)."""
import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _write(path, ts, ek, es, meta):
    with open(path, "w") as f:
        for t, a, b in zip(ts, ek, es):
            f.write(json.dumps({"t": t, "steps": 0, "E_k": a, "eps_S": b, "eps_D": 0.0, "eps_T": b}) + "\n")
        f.write(json.dumps(meta) + "\n")


def test_tgv_compare_deviations_and_svg(tmp_path):
    t = np.linspace(0.0, 10.0, 101)
    ek = 0.125 * np.exp(-0.2 * t)
    es = 0.01 * np.sin(np.pi * t / 10.0) + 0.001
    ref = tmp_path / "ref.jsonl"
    run = tmp_path / "run.jsonl"
    _write(ref, t, ek, es, {"scheme": "cgks5", "n": 64, "device_seconds_stepping": 10.0, "steps": 100})
    t2 = np.linspace(0.0, 10.0, 37)  # other sample times: the reference is interpolated
    _write(run, t2, np.interp(t2, t, ek) * 1.02, np.interp(t2, t, es) - 0.001,
           {"scheme": "gks2", "n": 128, "device_seconds_stepping": 25.0, "steps": 300})
    svg = tmp_path / "h.svg"
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tgv_compare.py"), str(ref), str(run),
                          "--svg", str(svg)], capture_output=True, text=True, check=True).stdout
    d = json.loads(out)
    r = d["runs"][0]
    assert r["run"] == "GKS-2nd 128^3" and d["reference"]["run"] == "CGKS-5th 64^3"
    assert r["E_k_max_abs_dev_rel"] == pytest.approx(0.02, rel=1e-3)  # 2 % of E_k(0) = max E_k
    assert r["eps_S_max_abs_dev_rel"] == pytest.approx(0.001 / es.max(), rel=1e-6)
    assert r["time_ratio_to_first_run"] == 1.0 and r["device_seconds"] == 25.0
    root = ET.parse(svg).getroot()
    assert sum(1 for e in root.iter() if e.tag.endswith("polyline")) == 4  # 2 runs x 2 panels


def test_bench_workload_names():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.make_case("tgv24").n == (24, 24, 24)
    c = bench.make_case("tgv_ss12")
    assert c.n == (12, 12, 12) and c.sutherland_S > 0 and c.nonlinear
    assert bench.make_case("hit16").n == (16, 16, 16)
    with pytest.raises(ValueError):
        bench.make_case("tgv")


def test_slab_inputs_tile_the_global_grid():
    # the per-rank inputs of the decomposed bench runs: slabs of tgv(n) concatenate to tgv(n)
    # (strong scaling), and the 512 x 512 x 64 blocks are the z-planes of the 512^3 TGV
    from cgks_inputs import tgv
    full = tgv(16)
    parts = [tgv(16, z0=4 * r, nzb=4) for r in range(4)]
    assert np.array_equal(np.concatenate([p.Q for p in parts], axis=1), full.Q)
    assert np.array_equal(np.concatenate([p.G for p in parts], axis=2), full.G)
    sys.path.insert(0, ROOT)
    import bench
    b = bench.slab512(8, 3)
    assert b.n == (512, 512, 512) and b.Q.shape == (5, 64, 512, 512)
    b1 = bench.slab512(1, 0)
    assert b1.n == (512, 512, 64) and b1.hi[2] - b1.lo[2] == pytest.approx(2 * np.pi / 8)


def test_pencil_inputs_tile_the_global_grid():
    # bench.py --strong --pencil PyxPz: the per-rank blocks (rank = ry + Py rz) tile tgv(n)
    from cgks_inputs import tgv
    from paper_2508_19911_b200.binding import decompose_pencil
    sys.path.insert(0, ROOT)
    import bench
    full = tgv(16)
    Q = np.zeros_like(full.Q)
    G = np.zeros_like(full.G)
    for r in range(8):
        b = bench.pencil_block(16, 2, 4, r)
        off, nl, _ = decompose_pencil((16, 16, 16), (1, 2, 4), r)
        assert b.n == (16, 16, 16) and b.Q.shape == (5, nl[2], nl[1], nl[0])
        Q[:, off[2]:off[2] + nl[2], off[1]:off[1] + nl[1]] = b.Q
        G[:, :, off[2]:off[2] + nl[2], off[1]:off[1] + nl[1]] = b.G
    assert np.array_equal(Q, full.Q) and np.array_equal(G, full.G)


def test_bench_reference_arm_line():
    # the reference arm (CPU oracle on a bounded sample) prints one JSON line with our arm's config
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "cell-updates/s" and line["higher_is_better"]
    assert line["config"]["workload"] == "tgv 128x128x128" and line["config"]["global_cells"] == 128 ** 3
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_bench_launch_plan():
    # --gpus N starts N ranks itself unless under a launcher; a mismatch is refused
    import bench
    what, argv = bench.launch_plan(4, {})
    assert what == "exec"
    assert "torch.distributed.run" in argv and "--nproc-per-node=4" in argv
    assert argv[argv.index("--master-addr") + 1] == "127.0.0.1"
    assert bench.launch_plan(1, {}) == ("run", None)
    assert bench.launch_plan(2, {"WORLD_SIZE": "2"}) == ("run", None)
    what, msg = bench.launch_plan(4, {"WORLD_SIZE": "2"})
    assert what == "refuse" and "WORLD_SIZE=2" in msg


def test_bench_gpus2_launches_two_ranks_cpu():
    # the launcher end to end on CPU: the reference arm under 2 gloo ranks; rank 0 alone prints the line
    import json
    import subprocess
    import sys
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["config"]["workload"] == "tgv 512x512x128"  # north_star weak scaling: 512 x 512 x 64 per GPU
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], capture_output=True,
                       text=True, timeout=60, env={**env, "WORLD_SIZE": "2"})
    assert r.returncode == 2 and "refusing" in r.stderr
