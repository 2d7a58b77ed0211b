"""Static validity of the tcgen05 halo row tiles (sketch 11, knobs BM, BN, STAGES, EPI, EW): stride-1,
undilated convs over whole 64-channel blocks; the shared-memory rule counts the STAGES staged
input rows and the resident weights.  Uses the handle-free catalogue query tuner_sketch_valid
(no device needed)."""
import itertools

from paper_2406_20037_b200 import sketch_space, sketch_valid

SK = 11


def _valid_halo(shape):
    sp = sketch_space(SK)
    return [list(v) for v in itertools.product(*sp) if sketch_valid("conv2d", shape, SK, v, "bf16")]


def base(**kw):
    s = {"N": 16, "H": 224, "W": 224, "C": 64, "K": 64, "R": 3, "S": 3, "stride": (1, 1), "pad": (1, 1),
         "dil": (1, 1)}
    s.update(kw)
    return s


def test_halo_valid_for_stride1_channel_blocks():
    pts = _valid_halo(base())
    assert pts
    assert all(v[2] >= 4 for v in pts)   # STAGES = row slots >= R + 1
    assert {v[0] for v in pts} == {128, 256}
    # smem: 1024 + STAGES * 17 KB rows + 9 taps * (BN / CG) * 128 B resident + 32 KB + 256 <= 227 KB
    assert [128, 64, 7, 1, 4] in pts       # 119 + 72 + 33 KB
    assert [128, 64, 8, 1, 4] not in pts   # 136 + 72 + 33 KB
    assert [256, 128, 7, 1, 8] in pts       # BN / CG = 64 rows of B per CTA
    assert [128, 128, 4, 1, 4] not in pts   # 68 + 144 + 33 KB
    assert not any(v[1] // (v[0] // 128) > 96 for v in pts)  # BM 256 x BN 192: 108 KB resident


def test_halo_rejected_off_its_domain():
    assert not _valid_halo(base(stride=(2, 2)))
    assert not _valid_halo(base(dil=(2, 2)))
    assert not _valid_halo(base(C=32))
    assert not _valid_halo(base(C=96))
    assert not _valid_halo(base(R=1, S=130, pad=(0, 0), W=300))  # window wider than a TMA box


def test_halo_two_channel_blocks_do_not_fit():
    # 2 channel blocks: >= 4 rows x 34 KB + 2 x 9 x 32 x 128 B resident + 33 KB > 227 KB
    assert not _valid_halo(base(C=128, K=128, H=56, W=56))
    assert _valid_halo(base(R=1, S=1, pad=(0, 0), C=128, K=64))  # 1x1: 2 slots x 34 KB + 2 x 8 KB


def test_sketch3_has_no_halo_tile():
    sp = sketch_space(3)
    assert sp[5] == [8, 16, 32]
    assert sketch_valid("conv2d", base(stride=(2, 2)), 3, [128, 64, 64, 4, 1, 16, 0, 0, 1, 4], "bf16")
