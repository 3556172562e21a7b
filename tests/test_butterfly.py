"""Host model of the transposing butterfly (`rowsum8` / `rowsum8_row` /
`owners_sum`, paper_1906_04051_b200/csrc/kernels.cuh) used by the 8-warp
power iteration of the Ritz harvest: 32 lanes each hold 8 partial row sums;
after 9 xor-shuffles lane l must hold the full sum of row
r(l) = 4 b4 + 2 b3 + b2, and the lanes l % 4 == 0 are the 8 row owners.
The model replays the kernel's exact shuffle/add sequence lane by lane."""
import numpy as np


def shfl_xor(vals, mask):
    return [vals[l ^ mask] for l in range(32)]


def rowsum8(a):
    # a: 32 lanes x 8 values
    b = [[0.0] * 4 for _ in range(32)]
    for q in range(4):
        send = [a[l][q] if l & 16 else a[l][q + 4] for l in range(32)]
        recv = shfl_xor(send, 16)
        for l in range(32):
            b[l][q] = (a[l][q + 4] if l & 16 else a[l][q]) + recv[l]
    c = [[0.0] * 2 for _ in range(32)]
    for q in range(2):
        send = [b[l][q] if l & 8 else b[l][q + 2] for l in range(32)]
        recv = shfl_xor(send, 8)
        for l in range(32):
            c[l][q] = (b[l][q + 2] if l & 8 else b[l][q]) + recv[l]
    send = [c[l][0] if l & 4 else c[l][1] for l in range(32)]
    recv = shfl_xor(send, 4)
    d = [(c[l][1] if l & 4 else c[l][0]) + recv[l] for l in range(32)]
    for mask in (2, 1):
        r = shfl_xor(d, mask)
        d = [d[l] + r[l] for l in range(32)]
    return d


def row_of(lane):
    return ((lane >> 2) & 1) | (((lane >> 3) & 1) << 1) | (((lane >> 4) & 1) << 2)


def owners_sum(v):
    for mask in (4, 8, 16):
        r = shfl_xor(v, mask)
        v = [v[l] + r[l] for l in range(32)]
    return v


def test_rowsum8_maps_every_lane_to_its_row_sum():
    rng = np.random.default_rng(3)
    a = rng.integers(-1000, 1000, size=(32, 8)).astype(float).tolist()  # exact in fp64
    d = rowsum8(a)
    col = np.asarray(a).sum(axis=0)
    for lane in range(32):
        assert d[lane] == col[row_of(lane)], lane
    owners = [l for l in range(32) if l % 4 == 0]
    assert sorted(row_of(l) for l in owners) == list(range(8))


def test_owners_sum_collects_the_eight_owner_lanes():
    rng = np.random.default_rng(4)
    v = rng.integers(-50, 50, size=32).astype(float)
    masked = [v[l] if l % 4 == 0 else 0.0 for l in range(32)]
    s = owners_sum(masked)
    assert s[0] == sum(v[l] for l in range(0, 32, 4))
