"""Host-side checks of the layer-wise parameter broadcast plan (CPU)."""
from paper_1707_09414_b200.params import layout, messages
from paper_1707_09414_b200.workloads import MODELS


def test_workload_sizes_match_survey_totals():
    # VGG-16 553,430,176 B in 32 tensors; AlexNet 244,403,360 B
    # in 16; ResNet-50 102,228,128 B in 161; LeNet 8 tensors.
    assert (len(MODELS["vgg16"]), sum(MODELS["vgg16"])) == (32, 553430176)
    assert (len(MODELS["alexnet"]), sum(MODELS["alexnet"])) == (16, 244403360)
    assert (len(MODELS["resnet50"]), sum(MODELS["resnet50"])) == (161, 102228128)
    assert MODELS["lenet"] == [2000, 80, 100000, 200, 1600000, 2000, 20000, 40]


def test_layout_and_buckets_cover_every_tensor():
    for name, sizes in MODELS.items():
        offs, total = layout(sizes)
        assert all(o % 256 == 0 for o in offs) and total >= sum(sizes)
        for bucket in (0, 1 << 16, 1 << 20, 64 << 20):
            msgs = messages(sizes, bucket)
            covered = set()
            for off, n in msgs:
                for o, s in zip(offs, sizes):
                    if off <= o and o + s <= off + n:
                        covered.add(o)
            assert covered == set(offs), (name, bucket)
            if bucket == 0:
                assert len(msgs) == len(sizes)
            else:
                assert all(n >= bucket for _, n in msgs[:-1])
