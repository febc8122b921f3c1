"""Ingest path (host code): PLY ascii / binary_little_endian
and XYZ readers and the selection-sampling subsample against the
reference's own read_cloud / subsample (oracle/_ref), on files written here:
extra vertex properties, list properties, extra elements, comments, CRLF,
and the error cases."""
import struct

import numpy as np
import pytest

from paper_1807_02587_b200 import treereg as tr


def _ref():
    try:
        from oracle.oracle import Ref
        return Ref()
    except (ImportError, FileNotFoundError):
        pytest.skip("reference oracle not built")


PTS = np.random.default_rng(7).normal(size=(257, 3)) * [1.0, 2.0, 0.5]


def _ply_ascii(path, pts):
    lines = ["ply", "format ascii 1.0", "comment made by tests", f"element vertex {len(pts)}",
             "property double x", "property float nx", "property double y", "property double z",
             "property uchar red", "element face 2", "property list uchar int vertex_indices",
             "end_header"]
    for p in pts:
        lines.append(f"{float(p[0])!r} 0.5 {float(p[1])!r} {float(p[2])!r} 7")
    lines += ["3 0 1 2", "4 0 1 2 3"]
    path.write_text("\r\n".join(lines) + "\r\n")


def _ply_binary(path, pts, f32=False):
    head = ["ply", "format binary_little_endian 1.0", "element info 1", "property list uchar float v",
            f"element vertex {len(pts)}", f"property {'float' if f32 else 'double'} x",
            f"property {'float' if f32 else 'double'} y", "property ushort s",
            f"property {'float' if f32 else 'double'} z", "end_header"]
    body = bytearray()
    body += struct.pack("<B2f", 2, 1.0, 2.0)
    for p in pts:
        fmt = "<f" if f32 else "<d"
        body += struct.pack(fmt, p[0]) + struct.pack(fmt, p[1]) + struct.pack("<H", 3)
        body += struct.pack(fmt, p[2])
    path.write_bytes(("\n".join(head) + "\n").encode() + bytes(body))


def _xyz(path, pts):
    lines = ["# comment", ""] + [f"  {float(p[0])!r}\t{float(p[1])!r} {float(p[2])!r}" for p in pts]
    path.write_text("\n".join(lines) + "\n")


@pytest.mark.parametrize("kind", ["ply_ascii", "ply_binary", "ply_binary_f32", "xyz"])
def test_reader_matches_reference(tmp_path, kind):
    ref = _ref()
    f = tmp_path / f"c.{kind}"
    if kind == "ply_ascii":
        _ply_ascii(f, PTS)
    elif kind == "ply_binary":
        _ply_binary(f, PTS)
    elif kind == "ply_binary_f32":
        _ply_binary(f, PTS, f32=True)
    else:
        _xyz(f, PTS)
    ours = tr.read_cloud(f)
    theirs = ref.read_cloud(f)
    assert ours.shape == theirs.shape == PTS.shape
    if kind == "ply_binary_f32":
        assert np.array_equal(ours, PTS.astype(np.float32).astype(np.float64))
    assert np.array_equal(ours, theirs)


@pytest.mark.parametrize("content", [
    b"plx\nformat ascii 1.0\n",
    b"ply\nformat binary_big_endian 1.0\nelement vertex 1\nproperty double x\nend_header\n",
    b"ply\nformat ascii 1.0\nelement vertex 1\nproperty double x\nproperty double y\nend_header\n1 2\n",
    b"ply\nformat ascii 1.0\nelement vertex 2\nproperty double x\nproperty double y\n"
    b"property double z\nend_header\n1 2 3\n",
    b"ply\nformat binary_little_endian 1.0\nelement vertex 1\nproperty double x\nproperty double y\n"
    b"property double z\nend_header\n\x00\x00",
    b"1 2 3\n4 5\n",
    b"1 2 3 4\n",
    b"1 2 nan\n",
])
def test_reader_errors_match_reference(tmp_path, content):
    ref = _ref()
    f = tmp_path / "bad"
    f.write_bytes(content)
    with pytest.raises(RuntimeError):
        tr.read_cloud(f)
    with pytest.raises(RuntimeError):
        ref.read_cloud(f)


def test_format_mismatch_and_missing_file(tmp_path):
    f = tmp_path / "a.ply"
    _ply_ascii(f, PTS[:5])
    with pytest.raises(RuntimeError):
        tr.read_cloud(f, "ply_binary")
    assert tr.read_cloud(f, "ply_ascii").shape == (5, 3)
    with pytest.raises(RuntimeError):
        tr.read_cloud(tmp_path / "missing.ply")


@pytest.mark.parametrize("n,m,seed", [(1000, 1, 3), (1000, 999, 4), (5000, 1234, 5), (7, 7, 0)])
def test_subsample_matches_reference(n, m, seed):
    ref = _ref()
    pts = np.random.default_rng(seed).normal(size=(n, 3))
    assert np.array_equal(tr.subsample(pts, m, seed), ref.subsample(pts, m, seed))
    with pytest.raises(tr.InvalidArgument):
        tr.subsample(pts, n + 1, seed)
