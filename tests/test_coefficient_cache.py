"""CPU: the coefficient-table on-disk format (reference
coefficients.cpp:113-214): serialize() is byte-identical to the reference's,
deserialize() accepts exactly what the reference accepts, and the
FKT_CACHE_DIR cache is read and written in the reference's file naming.
Host-only code (no GPU)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = [(2, 4), (3, 6), (3, 8), (5, 4), (7, 3), (3, 0), (2, 1), (4, 12), (3, 20)]


@pytest.mark.parametrize("d,p", SHAPES)
def test_serialize_matches_reference(fkt, ref, d, p):
    ours = fkt.coefficientTable(d, p).serialize()
    assert ours == ref.tbar_serialize(d, p)
    assert ours.startswith(f"fkt-tbar 1 {d} {p}\n")
    t = fkt.CoefficientTable.deserialize(ours)
    assert t is not None and t.dimension() == d and t.maxOrder() == p and t.equalsComputed
    assert ref.tbar_deserialize(ours) == 1


def _variants(text):
    lines = text.splitlines()
    k, j, m, num, den = lines[1].split()
    yield "bad magic", text.replace("fkt-tbar", "fkt-tbaz", 1)
    yield "bad version", text.replace("fkt-tbar 1", "fkt-tbar 2", 1)
    yield "d < 2", text.replace("fkt-tbar 1 3 6", "fkt-tbar 1 1 6", 1)
    yield "p > 32", text.replace("fkt-tbar 1 3 6", "fkt-tbar 1 3 33", 1)
    yield "missing entry", "\n".join(lines[:-1]) + "\n"
    yield "zero denominator", "\n".join([lines[0], f"{k} {j} {m} {num} 0"] + lines[2:]) + "\n"
    yield "bad index", "\n".join([lines[0], f"{k} {int(j) + 1} {m} {num} {den}"] + lines[2:]) + "\n"
    yield "empty", ""


def test_deserialize_rejects_like_reference(fkt, ref):
    text = ref.tbar_serialize(3, 6)
    for name, bad in _variants(text):
        assert fkt.CoefficientTable.deserialize(bad) is None, name
        assert ref.tbar_deserialize(bad) == -1, name
    # a valid but different table parses and compares unequal, in both
    lines = text.splitlines()
    k, j, m, num, den = lines[5].split()
    other = "\n".join(lines[:5] + [f"{k} {j} {m} {int(num) + 1} {den}"] + lines[6:]) + "\n"
    t = fkt.CoefficientTable.deserialize(other)
    assert t is not None and not t.equalsComputed
    assert ref.tbar_deserialize(other) == 0
    # non-normalised fractions are normalised on load (Rational(num, den))
    scaled = "\n".join([lines[0]] + [" ".join(l.split()[:3] + [str(3 * int(l.split()[3])), str(3 * int(l.split()[4]))])
                                     for l in lines[1:]]) + "\n"
    t = fkt.CoefficientTable.deserialize(scaled)
    assert t is not None and t.equalsComputed and ref.tbar_deserialize(scaled) == 1


CHILD = r"""
import sys
sys.path.insert(0, %r)
import paper_2106_04487_b200 as fkt
print(fkt.tbar(3, 6, int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]))[1])
""" % ROOT


def test_fkt_cache_dir_read_and_write(fkt, ref, tmp_path):
    env = dict(os.environ, FKT_CACHE_DIR=str(tmp_path / "cache"))
    f = tmp_path / "cache" / "fkt-tbar-v1-d3-p6.txt"
    out = subprocess.run([sys.executable, "-c", CHILD, "2", "4", "3"], env=env, check=True, capture_output=True,
                         text=True).stdout.strip()
    assert f.exists() and f.read_text() == ref.tbar_serialize(3, 6)  # written in the reference's format
    assert out == fkt.tbar(3, 6, 2, 4, 3)[1]
    # a valid cached table is what the process uses (plan persistence)
    lines = f.read_text().splitlines()
    idx = next(i for i, l in enumerate(lines[1:], 1) if l.split()[:3] == ["2", "4", "3"])
    k, j, m, num, den = lines[idx].split()
    lines[idx] = f"{k} {j} {m} 7 11"
    f.write_text("\n".join(lines) + "\n")
    out = subprocess.run([sys.executable, "-c", CHILD, "2", "4", "3"], env=env, check=True, capture_output=True,
                         text=True).stdout.strip()
    assert out == "7/11"
    # a corrupt file is ignored and rewritten
    f.write_text("garbage\n")
    out = subprocess.run([sys.executable, "-c", CHILD, "2", "4", "3"], env=env, check=True, capture_output=True,
                         text=True).stdout.strip()
    assert out == fkt.tbar(3, 6, 2, 4, 3)[1] and f.read_text() == ref.tbar_serialize(3, 6)
