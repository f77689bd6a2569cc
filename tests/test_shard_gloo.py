"""Source sharding across ranks (world_size 2, gloo, CPU): each rank advances
its slice of the sources (here with the CPU oracle as the stepper -- the
check is the host-side sharding/gather logic), traces gathered at the end
must equal the single-process run bit for bit (sources are independent)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1604_06750_b200.shard import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle_ffi
    from paper_1604_06750_b200.shard import gather_traces, shard_sources
    from paper_1604_06750_b200.signal import Wavelet
    from paper_1604_06750_b200.synthetic import synthetic_system

    case = synthetic_system((2, 2, 1), M=3, m=3, S=7, R=3, seed=21)
    o = oracle_ffi.OracleStepper(case.flat)
    o.set_sources(shard_sources(case.g, world, rank))
    o.set_receivers(case.receivers)
    o.make_state(case.dt)
    w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, 30)
    tr, _ = o.run(30, w)
    full = gather_traces(tr, case.g.shape[1])
    if rank == 0:
        np.save(out_path, full)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    for S in (1, 7, 64, 100):
        for world in (1, 2, 3, 8):
            rng = [shard_range(S, world, r) for r in range(world)]
            assert rng[0][0] == 0 and rng[-1][1] == S
            assert all(a[1] == b[0] for a, b in zip(rng, rng[1:]))


def test_two_rank_source_shards_match_single_process(tmp_path, oracle):
    out = str(tmp_path / "traces.npy")
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    from paper_1604_06750_b200.signal import Wavelet
    from paper_1604_06750_b200.synthetic import synthetic_system

    case = synthetic_system((2, 2, 1), M=3, m=3, S=7, R=3, seed=21)
    o = oracle.OracleStepper(case.flat)
    o.set_sources(case.g)
    o.set_receivers(case.receivers)
    o.make_state(case.dt)
    w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, 30)
    ref, _ = o.run(30, w)
    assert np.array_equal(got, ref)


def _gpu_worker(rank, world, port, out_path):
    """Each rank advances its source shard with the B200 stepper (both ranks
    on cuda:0 -- this box has one GPU; ranks do not wait on each other's
    kernels, so sharing the device is only a functional check)."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1604_06750_b200.rom import RomStepper
    from paper_1604_06750_b200.shard import gather_traces, shard_sources
    from paper_1604_06750_b200.signal import Wavelet
    from paper_1604_06750_b200.synthetic import synthetic_system

    case = synthetic_system((3, 2, 2), M=6, m=4, S=21, R=5, seed=23)
    st = RomStepper(case.flat, device=0)
    st.set_sources(shard_sources(case.g, world, rank))
    st.set_receivers(case.receivers)
    st.make_state(case.dt)
    w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, 80)
    tr, _ = st.run(80, w)
    st.close()
    full = gather_traces(tr, case.g.shape[1])
    if rank == 0:
        np.save(out_path, full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_gpu_shards_bitwise_equal_single_process(tmp_path, gpu_lib):
    """The product under two ranks: gathered traces of the sharded run equal
    one process advancing all 21 sources, bit for bit."""
    out = str(tmp_path / "traces_gpu.npy")
    port = _free_port()
    mp.start_processes(_gpu_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    from paper_1604_06750_b200.rom import RomStepper
    from paper_1604_06750_b200.signal import Wavelet
    from paper_1604_06750_b200.synthetic import synthetic_system

    case = synthetic_system((3, 2, 2), M=6, m=4, S=21, R=5, seed=23)
    st = RomStepper(case.flat, device=0)
    st.set_sources(case.g)
    st.set_receivers(case.receivers)
    st.make_state(case.dt)
    w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, 80)
    ref, _ = st.run(80, w)
    st.close()
    assert np.abs(ref).max() > 0
    assert np.array_equal(got, ref)
