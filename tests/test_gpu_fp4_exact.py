"""Exactness of the FP4 pair-sum GEMM (tcgen05 kind::mxf4 on E2M1 {0, 1}, fp32 accumulation in
TMEM) at large per-entry sums — VERDICT r01 "What's weak" 2 / ADVICE r01 (medium).

The claim under test (R14, include/cpi.h CPI_VARIANT_FP4): every S_ab entry is an
integer sum of 0/1 products, so an fp32 accumulator holds it exactly while it stays below 2^24,
whatever order the tensor core adds the 32-element block products in -- PROVIDED the hardware
keeps a full 24-bit significand while accumulating.  Earlier tensor cores accumulated
low-precision formats in fewer bits (Hopper FP8), so this is a hardware property that only a
measurement shows.  The largest sums any other test reaches are ~1.2k; here:

  * a 16 x 8 px layout (A = left 8x8, B = right 8x8) with N = 2^24 - 1 frames, the largest batch
    CPI_VARIANT_FP4 accepts: all-ones frames must give S_ab = N for every pair (24 significant
    bits), and dense random frames (P(bit) = 7/8) must match the kind::i8 path (int32 MMA
    accumulation, exact by construction) bit for bit and the closed-form row sums
    sum_q S_ab[p][q] = sum_i A^i_p n_B(i) (Eq. (1) numerators);
  * the paper's full 256x256 arms at N = 10^5 (BASELINE configs[2]) with all-ones, P = 7/8 and
    P = 1/2 frames: whole-matrix bit-equality with kind::i8, closed-form row / column sums, and
    sampled rows vs the CPU oracle.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

N_MAX = (1 << 24) - 1
SMALL_W, SMALL_H = 16, 8
SMALL_A, SMALL_B = (0, 0, 8, 8), (8, 0, 8, 8)


def _dense_bytes(shape, seed, ors=3):
    """Random bytes whose bits are 1 with probability 1 - 2^-ors (OR of `ors` fair bytes)."""
    rng = np.random.default_rng([synth.SEED_ARMS, seed])
    out = rng.integers(0, 256, size=shape, dtype=np.uint8)
    for _ in range(ors - 1):
        out |= rng.integers(0, 256, size=shape, dtype=np.uint8)
    return out


def _counts(frames, roi_a, roi_b, variant, width, height):
    from paper_2407_20692_b200 import Context
    n = frames.shape[0]
    ctx = Context(roi_a, roi_b, n, keep_counts=True, variant=variant, width=width, height=height)
    ctx.load_frames(frames)
    ctx.correlate(None)
    s_ab, s_a, s_b = ctx.counts_views()
    torch.cuda.synchronize()
    return ctx, s_ab, s_a, s_b


def _row_col_sums_np(frames, byte_a, byte_b, chunk=1 << 21):
    """Closed forms over the whole matrix for arms that are whole bytes of every frame row:
    row sums A^T n_B and column sums B^T n_A via the per-frame fired-pixel counts n_A(i), n_B(i),
    plus S_a, S_b (numpy, float64 BLAS in chunks; every partial sum < 2^53, so exact)."""
    n = frames.shape[0]
    row = col = sa = sb = 0.0
    for i0 in range(0, n, chunk):
        f = frames[i0:i0 + chunk]
        A = np.unpackbits(f[:, :, byte_a], axis=-1, bitorder="little").reshape(f.shape[0], -1).astype(np.float64)
        B = np.unpackbits(f[:, :, byte_b], axis=-1, bitorder="little").reshape(f.shape[0], -1).astype(np.float64)
        row = row + A.T @ B.sum(1)
        col = col + B.T @ A.sum(1)
        sa = sa + A.sum(0)
        sb = sb + B.sum(0)
    return tuple(np.asarray(x).astype(np.int64) for x in (row, col, sa, sb))


def test_fp4_all_ones_at_2p24_minus_1():
    """All-ones frames, N = 2^24 - 1: S_ab = S_a = S_b = N exactly (an fp32 accumulator with
    fewer than 24 significant bits cannot hold 2^24 - 1)."""
    frames = np.full((N_MAX, SMALL_H, SMALL_W // 8), 0xFF, dtype=np.uint8)
    ctx, s_ab, s_a, s_b = _counts(frames, SMALL_A, SMALL_B, "fp4", SMALL_W, SMALL_H)
    assert int(s_ab.min()) == N_MAX and int(s_ab.max()) == N_MAX
    assert int(s_a.min()) == N_MAX == int(s_b.max())
    ctx.close()


def test_fp4_dense_random_at_2p24_minus_1_matches_i8_and_closed_forms():
    frames = _dense_bytes((N_MAX, SMALL_H, SMALL_W // 8), seed=24)
    c4, s4, sa4, sb4 = _counts(frames, SMALL_A, SMALL_B, "fp4", SMALL_W, SMALL_H)
    got4, got_sa, got_sb = s4.cpu().numpy(), sa4.cpu().numpy(), sb4.cpu().numpy()
    c4.close()
    c8, s8, sa8, sb8 = _counts(frames, SMALL_A, SMALL_B, "tc", SMALL_W, SMALL_H)
    got8 = s8.cpu().numpy()
    c8.close()
    assert got4.min() > 12_000_000   # sums well above 2^23
    np.testing.assert_array_equal(got4, got8)
    row, col, sa, sb = _row_col_sums_np(frames, 0, 1)
    np.testing.assert_array_equal(got4.sum(1, dtype=np.int64), row)
    np.testing.assert_array_equal(got4.sum(0, dtype=np.int64), col)
    np.testing.assert_array_equal(got_sa, sa)
    np.testing.assert_array_equal(got_sb, sb)


ROWS = np.array([0, 255, 32768, 65535])


@pytest.mark.parametrize("kind", ["ones", "dense", "half"])
def test_fp4_fullsize_1e5_matches_i8_oracle_and_closed_forms(kind):
    """BASELINE configs[2] size (256^2 x 256^2, 10^5 frames) with dense data: per-entry sums up
    to 10^5 (all-ones), ~7.7e4 (P = 7/8) and ~2.5e4 (P = 1/2)."""
    n = 100_000
    shape = (n, 256, 64)
    if kind == "ones":
        frames = np.full(shape, 0xFF, dtype=np.uint8)
    elif kind == "dense":
        frames = _dense_bytes(shape, seed=25)
    else:
        frames = synth.bernoulli_frames(n, 0.5, seed=synth.SEED_ARMS)
    c4, s4, sa4, sb4 = _counts(frames, synth.ROI_FULL_A, synth.ROI_FULL_B, "fp4", 512, 256)
    c8, s8, _, _ = _counts(frames, synth.ROI_FULL_A, synth.ROI_FULL_B, "tc", 512, 256)
    assert torch.equal(s4, s8), "kind::mxf4 and kind::i8 pair sums differ"
    c8.close()
    if kind == "ones":
        assert int(s4.min()) == n == int(s4.max())
        c4.close()
        return
    row4 = s4.sum(1, dtype=torch.int64).cpu().numpy()
    col4 = s4.sum(0, dtype=torch.int64).cpu().numpy()
    got_rows = s4[torch.from_numpy(ROWS).cuda()].cpu().numpy()
    got_sa, got_sb = sa4.cpu().numpy(), sb4.cpu().numpy()
    c4.close()
    want = oracle.correlate(frames, synth.ROI_FULL_A, synth.ROI_FULL_B, rows=ROWS, threads=0)
    np.testing.assert_array_equal(got_rows, want["s_ab"])
    np.testing.assert_array_equal(got_sa, want["s_a"])
    np.testing.assert_array_equal(got_sb, want["s_b"])
    # closed forms from per-frame fired-pixel counts (chunked: the unpacked arms are 6.5 GB each)
    popc = np.array([bin(b).count("1") for b in range(256)], dtype=np.int64)
    n_a = popc[frames[:, :, 0:32]].sum(axis=(1, 2)).astype(np.float64)
    n_b = popc[frames[:, :, 32:64]].sum(axis=(1, 2)).astype(np.float64)
    row = np.zeros(65536, dtype=np.float64)
    col = np.zeros(65536, dtype=np.float64)
    ch = 2000
    for i0 in range(0, n, ch):
        A = np.unpackbits(frames[i0:i0 + ch, :, 0:32], axis=-1, bitorder="little").reshape(-1, 65536)
        row += n_b[i0:i0 + ch] @ A.astype(np.float64)
        B = np.unpackbits(frames[i0:i0 + ch, :, 32:64], axis=-1, bitorder="little").reshape(-1, 65536)
        col += n_a[i0:i0 + ch] @ B.astype(np.float64)
    np.testing.assert_array_equal(row4, row.astype(np.int64))
    np.testing.assert_array_equal(col4, col.astype(np.int64))
