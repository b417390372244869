"""Record JSONL I/O (reference proj/src/records.cpp:65-152): the C++
writer's lines are byte-identical to the oracle's restatement of nlohmann/json's dump, and
read_records -> to_line round-trips (NaN -> null -> NaN)."""
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_records_jsonl_bytes_match_oracle(tmp_path, G):
    from paper_2412_16490_b200 import _native as N
    from oracle import records_ref as R
    exe = tmp_path / "records_io"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'paper_2412_16490_b200/csrc/include'}",
                    str(ROOT / "tests/cpp/records_io.cpp"), str(N.LIB_PATH), f"-Wl,-rpath,{N.LIB_PATH.parent}",
                    "-o", str(exe)], check=True)
    out = tmp_path / "recs.jsonl"
    r = subprocess.run([str(exe), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = out.read_text().splitlines()
    assert len(lines) == 3
    for line in lines:
        obj = json.loads(line, parse_constant=lambda c: float(c))
        assert R.dump(obj) == line
    assert '"energy_total":null' in lines[1]
    assert '"seed":18446744073709551615' in lines[0]


def test_oracle_double_layout_kats():
    from oracle import records_ref as R
    cases = [(0.0, "0.0"), (-0.0, "-0.0"), (1.0, "1.0"), (0.1, "0.1"), (1e-4, "0.0001"), (1e-5, "1e-05"),
             (1234.5678, "1234.5678"), (1e14, "100000000000000.0"), (1e15, "1e+15"), (1e16, "1e+16"), (1e21, "1e+21"),
             (123456789012345.0, "123456789012345.0"), (1234567890123456.0, "1.234567890123456e+15"),
             (5e-324, "5e-324"), (1.7976931348623157e308, "1.7976931348623157e+308"),
             (0.30000000000000004, "0.30000000000000004"), (float("nan"), "null")]
    for v, s in cases:
        assert R.fmt_double(v) == s, (v, R.fmt_double(v), s)


NLOHMANN = Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty")


def test_records_and_oracle_layout_pinned_to_real_nlohmann(tmp_path, G):
    """The records writer's bytes and the oracle's restated double layout equal what the real
    nlohmann/json 3.11.3 (the reference's JSON library, records.cpp:65-152) dumps: each written
    line re-parsed and dumped by nlohmann comes back byte for byte, and json(v).dump() matches
    records_ref.fmt_double on the layout KATs and on 20000 random doubles."""
    import numpy as np
    import pytest
    from paper_2412_16490_b200 import _native as N
    from oracle import records_ref as R
    if not (NLOHMANN / "nlohmann" / "json.hpp").exists():
        pytest.skip("nlohmann header not in this image")
    dump = tmp_path / "nlohmann_dump"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{NLOHMANN}", str(ROOT / "tests/cpp/nlohmann_dump.cpp"), "-o",
                    str(dump)], check=True)
    exe = tmp_path / "records_io"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'paper_2412_16490_b200/csrc/include'}",
                    str(ROOT / "tests/cpp/records_io.cpp"), str(N.LIB_PATH), f"-Wl,-rpath,{N.LIB_PATH.parent}",
                    "-o", str(exe)], check=True)
    out = tmp_path / "recs.jsonl"
    assert subprocess.run([str(exe), str(out)], capture_output=True).returncode == 0
    ours = out.read_text().splitlines()
    theirs = subprocess.run([str(dump), str(out)], capture_output=True, text=True, check=True).stdout.splitlines()
    assert ours == theirs
    rng = np.random.default_rng(3)
    vals = [0.0, -0.0, 1.0, 0.1, 1e-4, 1e-5, 1234.5678, 1e14, 1e15, 1e16, 1e21, 123456789012345.0,
            1234567890123456.0, 5e-324, 1.7976931348623157e308, 0.30000000000000004, -2.5e-300]
    vals += list(rng.normal(size=10000) * 10.0 ** rng.integers(-30, 30, size=10000))
    vals += list(rng.uniform(-1, 1, size=10000))
    text = "\n".join(float(v).hex() for v in vals)
    got = subprocess.run([str(dump), "--doubles"], input=text, capture_output=True, text=True, check=True).stdout
    assert got.splitlines() == [R.fmt_double(float(v)) for v in vals]


def test_writer_double_layout_equals_real_nlohmann(tmp_path, G):
    """grasp::records::format_json_double (host/records.cpp, Grisu2 restated) equals the real
    nlohmann 3.11.3 json(v).dump() on 100000 doubles of every magnitude (the records' bytes)."""
    import numpy as np
    import pytest
    from paper_2412_16490_b200 import _native as N
    if not (NLOHMANN / "nlohmann" / "json.hpp").exists():
        pytest.skip("nlohmann header not in this image")
    dump = tmp_path / "nlohmann_dump"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{NLOHMANN}", str(ROOT / "tests/cpp/nlohmann_dump.cpp"), "-o",
                    str(dump)], check=True)
    ours = tmp_path / "json_double"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'paper_2412_16490_b200/csrc/include'}",
                    str(ROOT / "tests/cpp/json_double.cpp"), str(N.LIB_PATH), f"-Wl,-rpath,{N.LIB_PATH.parent}",
                    "-o", str(ours)], check=True)
    rng = np.random.default_rng(17)
    bits = rng.integers(0, 2 ** 63 - 1, size=50000, dtype=np.int64).view(np.float64)
    vals = np.concatenate([bits[np.isfinite(bits)], rng.normal(size=25000) * 10.0 ** rng.integers(-20, 20, 25000),
                           rng.uniform(-1, 1, 25000), [5e-324, 2.2250738585072014e-308, 1.7976931348623157e308]])
    text = "\n".join(float(v).hex() for v in vals)
    a = subprocess.run([str(ours)], input=text, capture_output=True, text=True, check=True).stdout
    b = subprocess.run([str(dump), "--doubles"], input=text, capture_output=True, text=True, check=True).stdout
    assert a.splitlines() == b.splitlines()
