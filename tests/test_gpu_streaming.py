"""GPU rqb_streaming (p/src/sketch.cpp:73-116) through the C ABI against the fp64 oracle's
restatement, mirroring the reference's own streaming tests (p/tests/test_sketch.cpp:143-181):
block-size independence and agreement with the in-memory rqb, the 2 + q pass count, plus the
RNMFMAT1 file source (FileColumnSource, p/src/data_io.cpp:185-223) and the error paths."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _opts(gpu, **kw):
    o = gpu.SketchOptions(target_rank=5, oversampling=10, power_iterations=2, seed=21)
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def test_block_size_independence_and_rqb_agreement(gpu, oracle):
    a = oracle.synth_lowrank(300, 200, 5, 0.0, 5)
    a /= np.linalg.norm(a)
    qm, bm = oracle.rqb(a, 5, 10, 2, seed=21)
    qb_mem = qm @ bm
    prev = None
    for bs in (1, 7, 64, 1024):
        r = gpu.rqb_streaming(a, _opts(gpu, block_size=bs))
        qb = r.q @ r.b
        assert np.linalg.norm(qb - qb_mem) <= 1e-10
        if prev is not None:
            assert np.linalg.norm(qb - prev) <= 1e-10
        prev = qb
        np.testing.assert_allclose(r.q.T @ r.q, np.eye(r.q.shape[1]), atol=1e-12)
        qo, bo = oracle.rqb_streaming(a, 5, 10, 2, seed=21, block_size=bs)
        np.testing.assert_allclose(qb, qo @ bo, atol=1e-12)


@pytest.mark.parametrize("q", [0, 1, 3])
def test_pass_count_is_two_plus_q(gpu, oracle, q):
    """p/tests/test_sketch.cpp:168-181: the source is read 2 + q times."""

    class CountingSource(gpu.ColumnSource):
        def __init__(self, a):
            self.src = gpu.MatrixColumnSource(a)
            self.columns_read = 0

        def rows(self):
            return self.src.rows()

        def cols(self):
            return self.src.cols()

        def read_columns(self, first, count, dst):
            self.columns_read += count
            self.src.read_columns(first, count, dst)

    a = oracle.synth_lowrank(60, 40, 3, 0.0, 2)
    src = CountingSource(a)
    gpu.rqb_streaming(src, gpu.SketchOptions(target_rank=3, oversampling=2, power_iterations=q, block_size=16, seed=6))
    assert src.columns_read == (2 + q) * a.shape[1]


def test_larger_streamed_sketch_matches_oracle(gpu, oracle):
    a = oracle.synth_lowrank(3000, 1100, 12, 0.05, 9)
    o = gpu.SketchOptions(target_rank=12, oversampling=8, power_iterations=2, seed=3, block_size=256)
    r = gpu.rqb_streaming(a, o)
    qo, bo = oracle.rqb_streaming(a, 12, 8, 2, seed=3, block_size=256)
    np.testing.assert_allclose(r.q @ r.b, qo @ bo, atol=1e-11 * np.abs(a).max())
    np.testing.assert_allclose(r.q @ r.q.T, qo @ qo.T, atol=1e-9)


def test_injected_omega_and_uniform_test_matrix(gpu, oracle):
    a = oracle.synth_lowrank(200, 150, 4, 0.1, 4)
    om = np.random.default_rng(1).standard_normal((150, 10))
    r = gpu.rqb_streaming(a, gpu.SketchOptions(target_rank=4, oversampling=6, power_iterations=1, block_size=33),
                          omega=om)
    qo, bo = oracle.rqb_streaming(a, 4, 6, 1, block_size=33, omega=om)
    np.testing.assert_allclose(r.q @ r.b, qo @ bo, atol=1e-12 * np.abs(a).max())
    r = gpu.rqb_streaming(a, gpu.SketchOptions(target_rank=4, oversampling=6, power_iterations=1, block_size=50,
                                               test_matrix=gpu.TestMatrixKind.Uniform, seed=8))
    qo, bo = oracle.rqb_streaming(a, 4, 6, 1, test_matrix=0, seed=8, block_size=50)
    np.testing.assert_allclose(r.q @ r.b, qo @ bo, atol=1e-12 * np.abs(a).max())


def test_file_source_matches_memory(gpu, oracle, tmp_path):
    a = oracle.synth_lowrank(257, 131, 5, 0.05, 12)
    path = tmp_path / "x.bin"
    gpu.write_matrix_bin(str(path), a)
    o = _opts(gpu, block_size=40)
    rf = gpu.rqb_streaming(gpu.FileColumnSource(str(path)), o)
    rm = gpu.rqb_streaming(a, o)
    assert np.array_equal(rf.q, rm.q) and np.array_equal(rf.b, rm.b)


def test_file_source_errors(gpu, tmp_path):
    o = _opts(gpu, block_size=16)
    with pytest.raises(gpu.IoError, match="cannot open"):
        gpu.rqb_streaming(gpu.FileColumnSource(str(tmp_path / "missing.bin")), o)
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTMAGIC" + b"\0" * 32)
    with pytest.raises(gpu.DataError, match='bad magic at byte 0 \\(expected "RNMFMAT1"\\)'):
        gpu.rqb_streaming(gpu.FileColumnSource(str(bad)), o)
    short = tmp_path / "short.bin"
    short.write_bytes(b"RNMFMAT1" + (10).to_bytes(8, "little") + (10).to_bytes(8, "little") + b"\0" * 80)
    with pytest.raises(gpu.DataError, match="file is 104 bytes, expected 824 for a 10x10 matrix"):
        gpu.rqb_streaming(gpu.FileColumnSource(str(short)), o)
    hdr = tmp_path / "hdr.bin"
    hdr.write_bytes(b"RNMFMAT1" + b"\0" * 4)
    with pytest.raises(gpu.DataError, match="truncated header"):
        gpu.rqb_streaming(gpu.FileColumnSource(str(hdr)), o)


def test_data_and_parameter_errors(gpu, oracle):
    a = oracle.synth_lowrank(100, 300, 4, 0.0, 1)
    a[7, 150] = np.nan
    with pytest.raises(gpu.DataError, match=r"rqb_streaming: non-finite values in columns \[128, 192\)"):
        gpu.rqb_streaming(a, _opts(gpu, target_rank=4, block_size=64))
    with pytest.raises(gpu.ParameterError, match="block size must be at least 1"):
        gpu.rqb_streaming(np.ones((10, 10)), _opts(gpu, target_rank=2, block_size=0))
    with pytest.raises(gpu.ParameterError, match="target rank"):
        gpu.rqb_streaming(np.ones((10, 10)), _opts(gpu, target_rank=11))

    class Failing(gpu.ColumnSource):
        def rows(self):
            return 20

        def cols(self):
            return 20

        def read_columns(self, first, count, dst):
            if first >= 10:
                raise gpu.IoError("disk gone")
            dst[:] = 1.0

    with pytest.raises(gpu.IoError, match="disk gone"):
        gpu.rqb_streaming(Failing(), _opts(gpu, target_rank=2, block_size=5))
