"""The offline data path (include/mel_dataset.h) on host cores: the file layout the
header documents (parsed here independently), the multi-threaded reader, and the epoch
order against oracle/dataset.py."""
import os
import struct

import numpy as np
import pytest

from mel_inputs import clients
from oracle import dataset as od
from paper_2309_16743_b200 import mel


@pytest.fixture(scope="module")
def lib():
    from paper_2309_16743_b200 import build
    build.build()
    return mel.load_library()


def _records(n_sims, tau, n):
    for s in range(n_sims):
        X = clients.client_X(s)
        for t in range(tau):
            yield s, t, X, clients.client_field(s, t, n).astype(np.float32)


def test_file_layout_and_reader(lib, tmp_path):
    n, path = 1000, str(tmp_path / "d.bin")
    recs = list(_records(3, 7, n))
    assert mel.write_dataset(path, n, recs) == 21
    raw = open(path, "rb").read()
    magic, version, n_field, count, stride, index_off, data_off = struct.unpack_from("<QIIQQQQ", raw, 0)
    assert raw[:8] == struct.pack("<Q", magic) and version == 1 and n_field == n and count == 21
    assert stride == 4096 and data_off == 4096 and index_off == data_off + count * stride
    for i, (s, t, X, f) in enumerate(recs):
        sim, tt = struct.unpack_from("<II", raw, index_off + 32 * i)
        assert (sim, tt) == (s, t)
        assert raw[index_off + 32 * i + 8:index_off + 32 * i + 28] == X.tobytes()
        assert raw[data_off + i * stride:data_off + i * stride + 4 * n] == f.tobytes()
    for threads in (1, 4):
        ds = mel.Dataset(path, threads=threads)
        assert ds.count == 21 and ds.n_field == n
        idx = np.array([20, 0, 5, 5, 13], np.uint32)
        sim, t, X, F = ds.read(idx)
        for k, i in enumerate(idx):
            s, tt, Xr, f = recs[i]
            assert (sim[k], t[k]) == (s, tt) and X[k].tobytes() == Xr.tobytes() and F[k].tobytes() == f.tobytes()
        with pytest.raises(mel.MelError):
            ds.read([21])
        ds.close()
    with pytest.raises(mel.MelError):
        mel.Dataset(str(tmp_path / "missing.bin"))
    open(str(tmp_path / "junk.bin"), "wb").write(b"x" * 8192)
    with pytest.raises(mel.MelError):
        mel.Dataset(str(tmp_path / "junk.bin"))


@pytest.mark.parametrize("n", [0, 1, 2, 17, 5000])
def test_epoch_order_matches_oracle(lib, n):
    for seed, epoch in ((1, 0), (1, 1), (123456789012, 7)):
        assert np.array_equal(mel.epoch_order(n, seed, epoch).astype(np.int64), od.epoch_order(n, seed, epoch))
