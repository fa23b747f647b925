"""Host logic of the ArrayInRow record harness (paper_2002_05599_b200.measure)
against the reference's record format (bench.py:25-75,192-240)."""

import io
import os
import subprocess
import sys
from pathlib import Path

import pytest

from paper_2002_05599_b200 import measure, registry
from paper_2002_05599_b200.errors import ConfigurationError

REF_SRC = Path("/root/reference/pkg/src")


def test_seed_sequence_matches_reference_rule():
    # state = master % (M - 1) + 1, then lcg_next per measure
    s = measure.SeedSequence(0)
    assert s.next_seed() == 48271 and s.next_seed() == 182605794
    big = measure.SeedSequence(2**64 - 1)
    first = (2**64 - 1) % (measure.LCG_MODULUS - 1) + 1
    assert big.next_seed() == first * 48271 % measure.LCG_MODULUS
    with pytest.raises(ConfigurationError):
        measure.SeedSequence(-1)


def test_seed_for_cell_and_default_count():
    assert measure.seed_for_cell(5, 8) == (5 ^ (8 * 0x9E3779B97F4A7C15)) % 2**64
    assert measure.default_number_of_arrays(8) == 32 * 2**20 // 128 + 1
    with pytest.raises(ConfigurationError):
        measure.default_number_of_arrays(0)


def test_array_in_row_validation_before_any_device_work():
    with pytest.raises(ConfigurationError):
        measure.array_in_row("SN Best 4CmS", 8, 10, 1, 1)  # 1280 B does not exceed the cache budget
    with pytest.raises(ConfigurationError):
        measure.array_in_row("SN Best 4CmS", 8, None, 0, 1)


def test_csv_round_trip_and_header():
    recs = [measure.MeasurementRecord("SN Best 4CmS", 8, i, 0.25 * i - 1.0, "nanos") for i in range(4)]
    text = measure.records_to_csv_text(recs)
    assert text.splitlines()[0] == ",".join(measure.CSV_HEADER)
    assert measure.read_records(io.StringIO(text)) == recs
    with pytest.raises(ConfigurationError):
        measure.read_records(io.StringIO("a,b\n"))
    with pytest.raises(ConfigurationError):
        measure.read_records(io.StringIO(""))


def test_labels_resolve_like_the_reference():
    label, spec = measure._resolve("SN Best 4CmS")
    assert label == "SN Best 4CmS" and spec == registry.spec_network("best", "4CmS")
    assert measure._resolve(spec)[0] == "SN Best 4CmS"


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference sources absent")
def test_reference_reader_accepts_our_csv(tmp_path):
    recs = [measure.MeasurementRecord("SN Best 4CmS", 16, i, 1.5 + i, "nanos") for i in range(3)]
    path = tmp_path / "air.csv"
    measure.write_records(path, recs)
    code = ("import sys; from netsort import bench; r = bench.read_records(sys.argv[1]); "
            "print(len(r), r[2].cost, r[0].sorter, r[0].timer_kind)")
    env = dict(os.environ, PYTHONPATH=str(REF_SRC), NETSORT_BACKEND="python")
    out = subprocess.run([sys.executable, "-c", code, str(path)], env=env, capture_output=True, text=True,
                         cwd=tmp_path)
    assert out.returncode == 0, out.stderr
    assert out.stdout.split() == ["3", "3.5", "SN", "Best", "4CmS", "nanos"]


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the driver's reference arm) prints one JSON
    line with the contract keys, on the host CPU (no GPU needed)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "1",
                        "--cpu-rows", "2048", "--ns", "2,5"], capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "arrays/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
