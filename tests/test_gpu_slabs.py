"""Row-slab decomposition (the multi-GPU path) on ONE device: N slab engines share the GPU and
exchange halos through the same buffers and the same three-step tick protocol a multi-GPU run
uses (peer copies here, NCCL send/recv in paper_1803_04782_b200/slabs.py).  The result must be
bit-identical to the oracle — i.e. to the undivided grid — for every N, because every tie-break of
the model is on pedestrian id, never on ownership."""
import numpy as np
import pytest

from oracle import oracle, shim
from tests import scenarios as sc

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


CASES = [
    ("desk64", 2), ("desk64", 4), ("closed-four", 2), ("closed-ped3", 2), ("linear-regulation", 2),
    ("linear-regulation", 3), ("wide-ragged", 3), ("field21", 2), ("ped5", 2), ("k16", 3), ("d0.9-eight-ped1", 4),
]


@pytest.mark.parametrize("name,slabs", CASES)
def test_slabs_equal_undivided_grid(product_lib, monkeypatch, name, slabs):
    monkeypatch.setenv("SFC_SLABS", str(slabs))
    text = sc.DESK64 if name == "desk64" else sc.EXTRA.get(name) or dict(sc.acceptance3_scenarios())[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for chunk in (1, 7, 22, 30):  # crosses rebuild points of every scenario that has them
        np.testing.assert_array_equal(gpu.run(chunk), cpu.run(chunk), err_msg=f"{name} x{slabs} moved")
        assert gpu.tick == cpu.tick
        np.testing.assert_array_equal(gpu.centers(), cpu.centers(), err_msg=f"{name} x{slabs} tick {gpu.tick} centres")
        np.testing.assert_array_equal(gpu.occupancy(), cpu.occupancy(), err_msg=f"{name} x{slabs} tick {gpu.tick} occupancy")
        for k in range(3):
            np.testing.assert_array_equal(bits(gpu.image(k)), bits(cpu.image(k)), err_msg=f"{name} x{slabs} image {k}")
    gpu.verify()


@pytest.mark.parametrize("name,slabs", [("desk64", 2), ("closed-four", 2), ("wide-ragged", 3), ("field21", 2),
                                        ("sparse-periodic", 3), ("sparse-closed", 2), ("sparse-field15", 2)])
@pytest.mark.parametrize("path", ["window", "scatter-list", "listwalk-list"])
def test_slabs_with_active_tile_list(product_lib, monkeypatch, name, slabs, path):
    """Slabs keep the tiles whose field region reaches into the halo rows permanently active (the
    neighbours' events arrive there as row copies, unseen by this slab's k-4) and list the rest."""
    monkeypatch.setenv("SFC_SLABS", str(slabs))
    monkeypatch.setenv("SFC_K5_PATH", path.split("-")[0])
    if path.endswith("-list"):
        monkeypatch.setenv("SFC_K5_ACTIVE_LIST", "1")
    text = sc.DESK64 if name == "desk64" else sc.EXTRA[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for chunk in (1, 7, 22):
        np.testing.assert_array_equal(gpu.run(chunk), cpu.run(chunk), err_msg=f"{name} x{slabs} moved")
        np.testing.assert_array_equal(gpu.centers(), cpu.centers(), err_msg=f"{name} x{slabs} tick {gpu.tick} centres")
        np.testing.assert_array_equal(gpu.occupancy(), cpu.occupancy(), err_msg=f"{name} x{slabs} tick {gpu.tick} occupancy")
        for k in range(3):
            np.testing.assert_array_equal(bits(gpu.image(k)), bits(cpu.image(k)), err_msg=f"{name} x{slabs} image {k}")


@pytest.mark.parametrize("name,slabs", [("desk64", 2), ("field21", 2), ("wide-ragged", 3), ("closed-four", 2), ("field35", 2)])
@pytest.mark.parametrize("lazy", ["0", "1"])
def test_slabs_with_field_kernel(product_lib, monkeypatch, name, slabs, lazy):
    """The large-field kernel on row slabs: its tiles count rows from the slab's first owned row and
    its regions read the neighbours' events from the halo rows."""
    monkeypatch.setenv("SFC_SLABS", str(slabs))
    monkeypatch.setenv("SFC_K5_PATH", "field")
    monkeypatch.setenv("SFC_K5_STRICT", "1")
    monkeypatch.setenv("SFC_K5_FIELD_LAZY", lazy)
    text = sc.DESK64 if name == "desk64" else sc.EXTRA[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for chunk in (1, 5, 9):
        np.testing.assert_array_equal(gpu.run(chunk), cpu.run(chunk), err_msg=f"{name} x{slabs} moved")
        np.testing.assert_array_equal(gpu.centers(), cpu.centers(), err_msg=f"{name} x{slabs} tick {gpu.tick} centres")
        np.testing.assert_array_equal(gpu.occupancy(), cpu.occupancy(), err_msg=f"{name} x{slabs} tick {gpu.tick} occupancy")
        for k in range(3):
            np.testing.assert_array_equal(bits(gpu.image(k)), bits(cpu.image(k)), err_msg=f"{name} x{slabs} image {k}")


def test_slab_halo_too_thin_is_a_config_error(product_lib, monkeypatch):
    monkeypatch.setenv("SFC_SLABS", "8")  # 24 rows / 8 = 3 owned rows < halo 4
    gpu = shim.Sim.from_scenario(product_lib, sc.SEQPAR24)
    with pytest.raises(shim.ShimError) as e:
        gpu.run(1)
    assert e.value.kind == "ConfigError" and "slab_halo" in e.value.message


# ---- the multi-process path: one rank per slab, torch.distributed halo exchange ---------------

def _rank_main(rank, world, port, text, ticks, out, seed_on_device=False):
    import os

    import torch.distributed as dist

    from paper_1803_04782_b200 import slabs
    from paper_1803_04782_b200 import socfield as sf

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)  # both ranks share GPU 0: halos bounce through the host
    try:
        cfg = sf.parse_scenario(text)
        state = sf.seed_population(cfg)
        # seed_on_device: the slab builds its occupancy rows and images itself (no whole-grid host state);
        # `state` is then only the download target of this test
        runner = slabs.SlabRunner(sf, cfg, None if seed_on_device else state, dist, rank, world, 0)
        assert runner.population == state.population
        moved = runner.run(ticks)
        runner.download(state)  # this rank's rows and pedestrians only
        eng = runner.engine
        rows = slice(eng.row0, eng.row0 + eng.rows)
        out[rank] = dict(moved=list(moved), rows=(eng.row0, eng.rows), occ=state.occupancy()[rows].copy(),
                         img=[state.image(k)[rows].copy() for k in ("dir-attractive", "dir-repulsive", "recurrent-repulsive")],
                         centers=state.centers())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world,seed_on_device", [("desk64", 2, False), ("closed-four", 2, False),
                                                       ("linear-regulation", 3, False), ("desk64", 2, True),
                                                       ("sparse-periodic", 3, True)])
def test_multi_process_slabs(name, world, seed_on_device):
    import socket

    import torch.multiprocessing as mp

    text = sc.DESK64 if name == "desk64" else sc.EXTRA[name]
    ticks = 23
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_rank_main, args=(world, port, text, ticks, out, seed_on_device), nprocs=world, join=True)
    cpu = oracle.OracleSim.from_scenario(text)
    moved = cpu.run(ticks)
    total = np.sum([np.array(out[r]["moved"]) for r in range(world)], axis=0)
    np.testing.assert_array_equal(total, moved)
    owned = np.zeros(cpu.population, bool)
    for r in range(world):
        o = out[r]
        rows = slice(o["rows"][0], o["rows"][0] + o["rows"][1])
        np.testing.assert_array_equal(o["occ"], cpu.occupancy()[rows])
        for k in range(3):
            np.testing.assert_array_equal(bits(o["img"][k]), bits(cpu.image(k)[rows]))
        truth = cpu.centers()
        mine = (truth[:, 1] >= o["rows"][0]) & (truth[:, 1] < o["rows"][0] + o["rows"][1])  # pedestrians this rank owns now
        np.testing.assert_array_equal(o["centers"][mine], truth[mine])
        owned |= mine
    assert owned.all()
