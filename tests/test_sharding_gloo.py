"""world_size-2 gloo test of the calibration sharding path (CPU): LPT split -> per-rank
compute -> one all-gather of packed records; the result must equal the single-rank one."""
import os
import pickle
import socket
import tempfile

import numpy as np
import torch.multiprocessing as mp

from paper_2605_21072_b200 import calibrate


def _costs():
    return [float(((i * 37) % 11) + 1) * (3 if i % 10 == 9 else 1) for i in range(40)]


def _compute(ids):
    """Deterministic per-layer work (stands in for the GPU pipeline; depends only on the id)."""
    out = []
    for i in ids:
        rng = np.random.default_rng(1000 + i)
        n = 8 + i % 5
        no = i % 3
        out.append(calibrate.LayerRecord(i, no, np.sort(rng.choice(64, no, replace=False)),
                                         float(rng.random()), i % 3, rng.random(3), rng.random(n),
                                         rng.random(n)))
    return out


def _worker(rank, world, port, path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    recs = calibrate.calibrate_model_sharded(_costs(), _compute, rank, world)
    with open(f"{path}.{rank}", "wb") as f:
        pickle.dump([r.pack() for r in recs], f)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_calibration_matches_single_rank():
    single = calibrate.calibrate_model_sharded(_costs(), _compute, 0, 1)
    assert [r.index for r in single] == list(range(40))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "recs")
        mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
        for rank in range(2):
            with open(f"{path}.{rank}", "rb") as f:
                got = pickle.load(f)
            assert len(got) == 40
            for a, b in zip(single, got):
                np.testing.assert_array_equal(a.pack(), b)


def _calib_compute(ids):
    out = []
    for i in ids:
        rng = np.random.default_rng(5000 + i)
        n, k = 3 + i % 4, 5 + i % 7
        res = calibrate.LayerCalibResult(f"layer{i}", rng.random(n), rng.random(n),
                                         rng.integers(-128, 128, (n, k)).astype(np.int8), rng.random(),
                                         rng.random(), rng.random(), rng.random(i % 5))
        out.append(calibrate.CalibRecord(i, res))
    return out


def _calib_worker(rank, world, port, path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    recs = calibrate.calibrate_model_sharded(_costs(), _calib_compute, rank, world,
                                             unpack=calibrate.unpack_calib_records)
    with open(f"{path}.{rank}", "wb") as f:
        pickle.dump([bytes(r.pack()) for r in recs], f)
    dist.destroy_process_group()


def test_sharded_adaround_records_match_single_rank():
    """The AdaRound (K7) layer results all-gathered as byte records (int8 codes, f64 scales and
    traces): world_size 2 over gloo equals world_size 1, slot by slot."""
    single = calibrate.calibrate_model_sharded(_costs(), _calib_compute, 0, 1)
    want = [bytes(r.pack()) for r in single]
    assert [r.index for r in single] == list(range(40))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "crecs")
        mp.spawn(_calib_worker, args=(2, _free_port(), path), nprocs=2, join=True)
        for rank in range(2):
            with open(f"{path}.{rank}", "rb") as f:
                assert pickle.load(f) == want
