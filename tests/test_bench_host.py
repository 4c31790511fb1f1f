"""Host-side helpers of bench.py (no GPU): the algorithmic byte count of the selection (SURVEY.md
8(d)) and the E3 bin choice of the KV-cache variant (reading Z13)."""
import bench


def test_select_bytes_sequential_closed_form():
    # sequential Alg 1: n r (d e + 24) + 4 n r (r - 1)  (the SURVEY 8(d) formula)
    n, d, r, e = 65536, 128, 256, 2
    assert bench.select_bytes(n, d, r, e) == n * r * (d * e + 24) + 4 * n * r * (r - 1)
    # the headline figure quoted in SURVEY 8(d): 21.8 GB
    assert abs(bench.select_bytes(n, d, r, e) / 1e9 - 21.8) < 0.1


def test_select_bytes_blocked_bookkeeping():
    # blocked: per block the K rows and the residual read + write, once the new F rows, and the F
    # prefix re-read at each block start (Fread = sum of block-start pivot counts)
    n, d, r, e = 65536, 128, 256, 2
    got = bench.select_bytes(n, d, r, e, nblocks=17, fread=2146)
    assert got == n * (17 * (d * e + 16) + 8 * r + 8 * 2146)
    assert abs(got / 1e9 - 1.5624) < 1e-3


def test_kv_bins():
    import bench

    # E3: B = r / 12 bins of rb = 12; 25 % of a 32K context minus the 64 retained tokens
    assert bench.kv_bins(8192 - 64) == 677
    assert bench.kv_bins(5) == 1
