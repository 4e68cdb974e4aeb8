"""Multi-GPU readiness of the calibration sharding (config 4) on one GPU:
  * the real CalibrationShard (K3 -> K5 -> K4 on device) run for every rank's LPT share at
    G = 2 / 4 / 8, one rank after another, gives the G = 1 records byte for byte;
  * two processes sharing cuda:0 run their real shards and all-gather the packed records over
    torch.distributed (gloo): identical to G = 1;
  * the C++ driver (qarvd_calibrate_sharded: one host thread per rank, NCCL all-gather when the
    ranks' devices are distinct) gives the same records at world 1 (NCCL communicator over the
    GPU) and 2 / 4 / 8 (ranks sharing the GPU, host gather)."""
import os
import pickle
import socket
import tempfile

import numpy as np
import pytest
import torch

from paper_2605_21072_b200 import calibrate, synth

pytestmark = pytest.mark.gpu

FRAMES, ROWS = 21, 96


def _specs():
    return synth.wan_registry(blocks=2)  # 20 layers: K = 1536 / 8960, N = 1536 / 8960, text-token k/v


def _costs(specs):
    rows_of = lambda s: ROWS if s.tokens != synth.WAN_TEXT_LEN else synth.WAN_TEXT_LEN
    return [calibrate.layer_cost_bytes(s, FRAMES, rows_of(s)) for s in specs]


def _run_share(specs, ids):
    if not ids:
        return []
    w = calibrate.weighting_strategy("heuristic_exp", FRAMES)
    shard = calibrate.CalibrationShard(specs, ids, FRAMES, ROWS, frame_weights=w)
    shard.setup()
    return shard.run()


def _packed(recs):
    return calibrate.pack_records(sorted(recs, key=lambda r: r.index)).tobytes()


@pytest.fixture(scope="module")
def single(cuda):
    specs = _specs()
    return _packed(_run_share(specs, list(range(len(specs)))))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_real_shards_union_equals_single_rank(single, world):
    specs = _specs()
    assign = calibrate.lpt_assign(_costs(specs), world)
    assert sorted(i for a in assign for i in a) == list(range(len(specs)))
    recs = []
    for rank in range(world):
        recs += _run_share(specs, assign[rank])
    assert _packed(recs) == single


def _worker(rank, world, port, path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    specs = _specs()
    recs = calibrate.calibrate_model_sharded(_costs(specs), lambda ids: _run_share(specs, ids), rank, world)
    with open(f"{path}.{rank}", "wb") as f:
        pickle.dump(_packed(recs), f)
    dist.destroy_process_group()


def test_two_processes_real_shards_allgather(single):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "recs")
        mp.spawn(_worker, args=(2, port, path), nprocs=2, join=True)
        for rank in range(2):
            with open(f"{path}.{rank}", "rb") as f:
                assert pickle.load(f) == single


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_native_cpp_driver_matches(single, world):
    w = calibrate.weighting_strategy("heuristic_exp", FRAMES)
    recs, ms, used_nccl = calibrate.calibrate_sharded_native(_specs(), FRAMES, ROWS, world, devices=[0] * world,
                                                             frame_weights=w)
    assert used_nccl == (world == 1)  # one communicator over the GPU at world 1; shared device: host gather
    assert ms > 0
    assert _packed(recs) == single
