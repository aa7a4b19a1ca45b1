"""Row digest of ab_get_list_digest / oracle.compute_digest written out in numpy (tests only):
h = mix(((u64)(u32)i << 32 | (u32)j) ^ mix((sx+128) << 16 | (sy+128) << 8 | (sz+128))), mix = the
splitmix64 finaliser; digest = (rows, sum h mod 2^64, xor h).  Used to pin both implementations on
lists small enough to return as rows."""
import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix(z):
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def digest(rows):
    rows = np.asarray(rows, dtype=np.int64).reshape(-1, 5)
    a = (rows[:, 0].astype(np.uint64) << np.uint64(32)) | (rows[:, 1].astype(np.uint64) & np.uint64(0xFFFFFFFF))
    b = ((rows[:, 2] + 128).astype(np.uint64) << np.uint64(16)) | ((rows[:, 3] + 128).astype(np.uint64) << np.uint64(8)) \
        | (rows[:, 4] + 128).astype(np.uint64)
    h = mix(a ^ mix(b))
    s = int(np.sum(h, dtype=np.uint64)) if len(h) else 0
    x = int(np.bitwise_xor.reduce(h)) if len(h) else 0
    return (len(rows), s, x)
