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
