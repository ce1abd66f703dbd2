"""Deep-CNN chains (BASELINE config c5) on the planner side, no GPU: shape
validation, the byte model the ledger bills, and the reference's closed-form
swap volumes (W = 3|W|, K = 2|K| for PP at N=1) on the full
ResNet-1026 / VGG-416 shapes."""

import pytest

import paper_2202_01306_b200 as H
from paper_2202_01306_b200.cnn import CNN_PRESETS, CNNSpec, CONV, DOWN, HEAD, RES, cnn_profiles


def test_presets_match_their_names():
    convs = {k: sum(1 if t in (CONV, DOWN) else 2 if t == RES else 0 for t, *_ in s.layers)
             for k, s in CNN_PRESETS.items()}
    assert convs["resnet-1026"] == 1026
    assert convs["vgg-416"] == 416
    assert CNN_PRESETS["resnet-1026"].layers[-1] == (HEAD, 512, 0, 7, 7)


def test_shape_validation():
    with pytest.raises(ValueError):
        CNNSpec(((CONV, 64, 64, 8, 8), (RES, 64, 128, 8, 8), (HEAD, 128, 0, 8, 8)), 10)  # res changes width
    with pytest.raises(ValueError):
        CNNSpec(((DOWN, 64, 64, 8, 8), (HEAD, 64, 0, 8, 8)), 10)  # pooled output is 4x4
    with pytest.raises(ValueError):
        CNNSpec(((CONV, 3, 64, 8, 8), (HEAD, 64, 0, 8, 8)), 10)  # image must be padded to 64 channels


@pytest.mark.parametrize("name", ["resnet-1026", "vgg-416"])
def test_ledger_closed_forms_full_size(name):
    spec = CNN_PRESETS[name]
    prof = cnn_profiles(spec)
    R = spec.n_layer
    W = sum(4 * spec.layer_params(L) for L in range(R))
    mach = H.MachineModel(gpu_count=1, gpu_mem_capacity=64 << 30, pcie_bandwidth=55_000_000_000)
    step = R // 8
    packs = tuple((i, min(i + step, R) - 1) for i in range(0, R, step))
    cfg = H.Configuration(8, packs, 8, packs, 32, H.Mode.PP)
    g = H.generate_task_graph(cfg, mach, prof)
    sim = H.simulate(g, mach, prof)
    vol = sim.tensor_volumes
    assert vol["W"]["cpu_gpu_swap"] == 3 * W
    assert vol["K"]["cpu_gpu_swap"] == 2 * 2 * W
    heads = [lo for lo, _ in packs[:-1]]
    assert vol["sX"]["message_passing"] == 2 * 32 * sum(spec.x_bytes(L) for L in heads)


def test_fine_resnet_relays_in_plan():
    """Convolution-granularity ResNet: each block's skip edge becomes a relay
    annotation (serialize_graph); relays crossing a pack boundary appear as X /
    dY entries with src_layer -- zero-byte SHARED_MEMORY on one GPU, billed
    y(src) on the P2P channel when the packs sit on different GPUs
    (taskgraph.py:195-208)."""
    spec = CNN_PRESETS["resnet-fine-tiny"]
    chain = spec.chain()
    assert [(a.source, a.destination) for a in chain.relay_annotations] == [(0, 2), (2, 4), (5, 7), (7, 9)]
    prof = cnn_profiles(spec)
    pf, pb = ((0, 1), (2, 5), (6, 10)), ((0, 3), (4, 5), (6, 10))
    cfg = H.Configuration(2, pf, 2, pb, 8, H.Mode.PP)
    one = H.MachineModel(gpu_count=1, gpu_mem_capacity=8 << 30, pcie_bandwidth=55_000_000_000)
    g1 = H.generate_task_graph(cfg, one, prof, chain)
    relays = [(t.index, L, ch.src_layer, ch.kind.value) for t in g1.tasks for ents in t.inputs.values()
              for L, ch in ents.items() if ch.src_layer is not None]
    assert relays == [(1, 0, 0, "shared_memory"), (7, 2, 2, "shared_memory")]
    assert "peer2peer" not in {r[4] for r in H.simulate(g1, one, prof).ledger}
    two = H.MachineModel(gpu_count=2, gpu_mem_capacity=8 << 30, pcie_bandwidth=55_000_000_000)
    g2 = H.generate_task_graph(cfg, two, prof, chain)
    p2p = H.simulate(g2, two, prof).channel_volumes.get("peer2peer", {})
    assert p2p  # trunk and relay hand-offs between the two GPUs are billed
