"""The `sigker` command-line tool (reference tools/main.cpp, csv.cpp,
datagen.cpp, validate.cpp) on the B200 engine.

CPU: the generators are bit-identical to the reference's (tests/golden/
datagen.json, written by the reference itself), CSV parsing follows the
reference's grammar and error contract, usage errors exit 2.  GPU: kernel /
grid / gram / bench outputs and the validate suites, including the
fault-injection negative control (the suite must FAIL with exit code 4)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2502_20392_b200", "sigker")
GOLD = os.path.join(ROOT, "tests", "golden")


def run(*args, cwd=None, timeout=600):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=timeout, cwd=cwd)


def parse(text):
    return np.array([[float(c) for c in line.split(",")] for line in text.strip().splitlines()])


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(CLI):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2502_20392_b200", "csrc")], check=True)
    assert os.path.exists(CLI)


def test_usage_and_unknown_subcommand():
    assert run().returncode == 2
    assert run("--help").returncode == 0
    r = run("frobnicate")
    assert r.returncode == 2 and "unknown subcommand" in r.stderr


def test_gen_brownian_bit_identical_to_reference():
    g = json.load(open(os.path.join(GOLD, "datagen.json")))
    for c in g["brownian"]:
        if c["length"] > 1000:
            continue
        r = run("gen", "--kind", "brownian", "--len", c["length"], "--dim", c["dim"], "--seed", c["seed"])
        assert r.returncode == 0, r.stderr
        b = parse(r.stdout)
        assert b.shape == (c["length"], c["dim"])
        assert b[:3].ravel()[: len(c["first"])].tolist() == c["first"]
        assert b[-1].tolist() == c["last"]
        assert float(b.sum()) == c["sum"]


def test_gen_fbm_bit_identical_to_reference():
    g = json.load(open(os.path.join(GOLD, "datagen.json")))
    for c in g["fbm"]:
        r = run("gen", "--kind", "fbm", "--len", c["length"], "--dim", c["dim"], "--hurst", c["hurst"],
                "--seed", c["seed"])
        assert r.returncode == 0, r.stderr
        b = parse(r.stdout)
        assert b[-1].tolist() == c["last"]
        assert float(b.sum()) == c["sum"]


def test_gen_to_file_and_near_periodic(tmp_path):
    out = tmp_path / "np.csv"
    r = run("gen", "--kind", "near-periodic", "--len", 9, "--dim", 3, "--noise", 0.01, "--out", out)
    assert r.returncode == 0 and "-> " in r.stdout
    v = parse(out.read_text())
    assert v.shape == (9, 3) and np.all(np.abs(v) < 1.1)
    assert run("gen", "--kind", "spiral").returncode == 2


@pytest.mark.parametrize("content,needle", [
    ("1,2\n3\n", "ragged row 2"),
    ("1,2\n3,x\n", "non-numeric cell at row 2, column 2"),
    ("1,2\n3,inf\n", "non-finite value at row 2, column 2"),
    ("a,b\n", "no data rows"),
    ("\n1,2\nx,y\n", "non-numeric cell at row 3, column 1"),
])
def test_csv_parse_errors_exit_2(tmp_path, content, needle):
    bad = tmp_path / "bad.csv"
    bad.write_text(content)
    good = tmp_path / "good.csv"
    good.write_text("t,x\n0,0\n1,1\n")
    r = run("kernel", bad, good)
    assert r.returncode == 2, r
    assert "input error" in r.stderr and needle in r.stderr, r.stderr


def test_order_and_tol_are_exclusive(tmp_path):
    p = tmp_path / "a.csv"
    p.write_text("0\n1\n")
    r = run("kernel", p, p, "--order", 8, "--tol", 1e-9)
    assert r.returncode == 2 and "mutually exclusive" in r.stderr
    cfg = tmp_path / "c.json"
    cfg.write_text('{"order": 8, "tol": 1e-9}')
    assert run("kernel", p, p, "--config", cfg).returncode == 2
    cfg.write_text("[1, 2]")
    assert run("kernel", p, p, "--config", cfg).returncode == 2


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_kernel_unit_tile_prints_library_bits(tmp_path):
    """test_cli.cpp:73-88: K of the unit tile at order 24 is I0(2) to the printed digits."""
    p = tmp_path / "unit.csv"
    p.write_text("x\n0\n1\n")
    r = run("kernel", p, p, "--order", 24, "--json")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0].startswith("K=")
    assert abs(float(lines[0][2:]) - 2.2795853023360673) < 1e-13
    meta = json.loads(lines[1])
    assert meta["order"] == 24 and meta["tiles"] == 1 and meta["schema"] == 1


@pytest.mark.gpu
def test_kernel_adaptive_grid_and_padding(tmp_path):
    x, y = tmp_path / "x.csv", tmp_path / "y.csv"
    assert run("gen", "--len", 40, "--dim", 2, "--seed", 3, "--out", x).returncode == 0
    assert run("gen", "--len", 25, "--dim", 2, "--seed", 4, "--out", y).returncode == 0
    grid = tmp_path / "grid.csv"
    r = run("kernel", x, y, "--tol", 1e-12, "--grid", grid)
    assert r.returncode == 0, r.stderr
    k = float(r.stdout.split("=")[1])
    g = parse(grid.read_text())
    assert g.shape == (40, 40)  # both padded to the common length
    assert np.all(g[0] == 1.0) and np.all(g[:, 0] == 1.0)
    assert abs(g[-1, -1] - k) < 1e-12 * max(1, abs(k))


@pytest.mark.gpu
def test_gram_matrix_and_metadata(tmp_path):
    d = tmp_path / "fam"
    d.mkdir()
    for s in range(4):
        assert run("gen", "--len", 33, "--dim", 2, "--seed", s + 1, "--out", d / f"s{s}.csv").returncode == 0
    out = tmp_path / "g.csv"
    r = run("gram", d, "--out", out, "--tol", 1e-12, "--bound")
    assert r.returncode == 0, r.stderr
    m = parse(out.read_text())
    assert m.shape == (4, 4) and np.allclose(m, m.T, rtol=0, atol=0)
    meta = json.loads((tmp_path / "g.json").read_text())
    assert meta["size"] == 4 and meta["policy"] == "adaptive" and meta["failures"] == []
    assert len(meta["inputs"]) == 4 and "bound" in meta and meta["max_abs_increment_product"] > 0
    # same entries as the library's Gram on the same family
    from paper_2502_20392_b200 import sigker as sk
    fam = [parse((d / f"s{s}.csv").read_text()) for s in range(4)]
    lib = sk.gram_matrix(fam, sk.GramOptions(policy=sk.TruncationPolicy.adaptive(1e-12)))
    assert np.asarray(lib.values).reshape(4, 4).tolist() == m.tolist()


@pytest.mark.gpu
def test_validate_all_suites_pass():
    r = run("validate", "--suite", "all", timeout=1200)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln and not ln.startswith(" ")]
    assert [ln.split()[0] for ln in lines] == ["closed-form", "oracle-triangle", "bound", "invariance"]
    assert all(ln.endswith("PASS") for ln in lines)


@pytest.mark.gpu
def test_validate_fault_injection_is_caught():
    """Negative control (validate.cpp:17-25): flipping W[1][1] on the device must fail the suite."""
    r = run("validate", "--suite", "closed-form", "--inject-fault")
    assert r.returncode == 4, r.stdout
    assert "FAIL" in r.stdout


@pytest.mark.gpu
def test_bench_table(tmp_path):
    out = tmp_path / "b.csv"
    r = run("bench", "--lengths", 33, 65, 129, "--dims", 2, "--repeats", 2, "--oracle-max-len", 100, "--out", out)
    assert r.returncode == 0, r.stderr
    rows = out.read_text().strip().splitlines()
    assert rows[0] == "length,dim,order,mean_seconds,stdev_seconds,peak_live_series,mape"
    assert len(rows) == 4
    for row in rows[1:3]:
        cells = row.split(",")
        assert float(cells[6]) < 1e-6  # order 7 vs the depth-20 levelwise oracle on short Brownian paths
    assert rows[3].endswith(",")  # above --oracle-max-len: no accuracy cell


def test_validate_oracles_agree_with_the_restatement(tmp_path, restatement):
    """The CPU oracles behind `validate --suite oracle-triangle` (signature
    tensors, levelwise truncation, finite differences, Picard) reproduce the
    restated reference solver (oracle/, order 24) on random walks."""
    exe = os.path.join(ROOT, "build", "oracle_values")
    pkg = os.path.join(ROOT, "paper_2502_20392_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "oracle_values.cpp"), "-o", exe, "-L", pkg, "-lsigker",
                    "-lsigker_b200", f"-Wl,-rpath,{pkg}"], check=True)
    rng = restatement.rng(99)
    for k in range(6):
        n = 3 + k
        x = rng.random_series(n, 2, 0.8)
        y = rng.random_series(n + 1, 2, 0.8)
        fx, fy = tmp_path / "x.csv", tmp_path / "y.csv"
        np.savetxt(fx, x, delimiter=",", fmt="%.17g")
        np.savetxt(fy, y, delimiter=",", fmt="%.17g")
        out = subprocess.run([exe, fx, fy], capture_output=True, text=True, check=True).stdout.split()
        sig, lw, fd, pic = map(float, out)
        want = restatement.propagate(x, y, 24)[0]
        assert abs(sig - want) / abs(want) < 1e-8
        assert abs(lw - sig) / abs(sig) < 1e-12
        assert abs(fd - want) / abs(want) < 1e-4
        assert abs(pic - want) / abs(want) < 1e-2


@pytest.mark.gpu
def test_kernel_config_file_and_flag_override(tmp_path):
    """--config supplies option values; a flag given on the command line wins
    (tools/main.cpp:58-68)."""
    p = tmp_path / "unit.csv"
    p.write_text("0\n1\n")
    cfg = tmp_path / "c.json"
    cfg.write_text('{"order": 3}')
    r = run("kernel", p, p, "--config", cfg, "--json")
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout.strip().splitlines()[1])["order"] == 3
    assert abs(float(r.stdout.split("=")[1].split()[0]) - (1 + 1 + 1 / 4 + 1 / 36)) < 1e-15
    r = run("kernel", p, p, "--config", cfg, "--order", 24)
    assert abs(float(r.stdout.split("=")[1]) - 2.2795853023360673) < 1e-13
