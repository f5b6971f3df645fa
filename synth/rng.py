"""Counter-based leaf-value generator shared by the oracle and the CUDA path.

This module is INPUT GENERATION ONLY: it holds none of the method's arithmetic
(no contraction, no schedule, no memory model).  The CUDA library carries an
independent implementation of the same generator (csrc/kernels/trace.cu,
`fill_synthetic_kernel`, entry point `cc_fill_synthetic`); a GPU test checks the two bit for bit.  The
recipe is DESIGN.md §"Input recipe":

  key(seed, leaf)   = splitmix64(splitmix64(seed) XOR leaf)
  u(seed, leaf, j)  = (splitmix64(key + j) >> 11) * 2^-53          j = 2*e + part
  phase-limited  re = (0.75 + 0.5*u(2e)) * sigma
                 im = ((0.5*u(2e+1) - 0.25) * 0.5) * sigma          |phase| <= 9.5 deg
  random-phase   re = (2*u(2e) - 1) * sigma,  im = (2*u(2e+1) - 1) * sigma

where e is the flat complex-element index of the leaf in its [Lt, ...] row-major
layout (t outermost), so any time-slice range can be generated on its own.
sigma = 1/N for meson leaves and 1/sqrt(S*N^3) for baryon leaves, which keeps
every node O(sigma) through MM1/BM1/BB2 and every trace O(1).

All arithmetic is uint64 modular (numpy wraps) and IEEE double with one
rounding per operation; the CUDA side uses the same operations with explicit
round-to-nearest intrinsics, so the values agree bit for bit.
"""
import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

MODE_PHASE_LIMITED = 0
MODE_RANDOM_PHASE = 1


def splitmix64(x):
    """SplitMix64 finaliser of (x + golden); x is a numpy uint64 scalar or array."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def leaf_key(seed, leaf_id):
    return splitmix64(splitmix64(np.uint64(seed)) ^ np.uint64(leaf_id))


def uniforms(seed, leaf_id, j0, count):
    """u(seed, leaf, j) for j in [j0, j0+count) as float64 in [0, 1)."""
    key = leaf_key(seed, leaf_id)
    with np.errstate(over="ignore"):
        j = np.arange(count, dtype=np.uint64) + np.uint64(j0)
        bits = splitmix64(key + j)
    return (bits >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def meson_sigma(N):
    return 1.0 / float(N)


def baryon_sigma(N, S):
    return 1.0 / np.sqrt(float(S * N ** 3))


def leaf_values(seed, leaf_id, e0, count, sigma, mode=MODE_PHASE_LIMITED):
    """complex128 values of elements [e0, e0+count) of one leaf."""
    u = uniforms(seed, leaf_id, 2 * e0, 2 * count)
    u1 = u[0::2]
    u2 = u[1::2]
    out = np.empty(count, dtype=np.complex128)
    if mode == MODE_PHASE_LIMITED:
        out.real = (0.75 + 0.5 * u1) * sigma
        out.imag = ((0.5 * u2 - 0.25) * 0.5) * sigma
    elif mode == MODE_RANDOM_PHASE:
        out.real = (2.0 * u1 - 1.0) * sigma
        out.imag = (2.0 * u2 - 1.0) * sigma
    else:
        raise ValueError("unknown mode %r" % (mode,))
    return out


def leaf_tensor(seed, leaf_id, shape, sigma, mode=MODE_PHASE_LIMITED, t_range=None):
    """Whole leaf (or the time slices t_range=(t0,t1)) as a complex128 array of `shape`."""
    per_t = int(np.prod(shape[1:]))
    t0, t1 = (0, shape[0]) if t_range is None else t_range
    vals = leaf_values(seed, leaf_id, t0 * per_t, (t1 - t0) * per_t, sigma, mode)
    return vals.reshape((t1 - t0,) + tuple(shape[1:]))


def leaf_values_into(out, seed, leaf_id, e0, sigma, mode=MODE_PHASE_LIMITED, chunk=1 << 22, workers=None):
    """leaf_values(seed, leaf_id, e0, out.size, sigma, mode) written into the complex128 array
    `out` in chunks on a thread pool (numpy releases the GIL in its loops): the same values,
    for multi-GiB leaves at full config sizes."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    flat = out.reshape(-1)
    n = flat.size
    workers = workers or max(1, min(32, len(os.sched_getaffinity(0))))

    def work(a):
        b = min(n, a + chunk)
        flat[a:b] = leaf_values(seed, leaf_id, e0 + a, b - a, sigma, mode)
    with ThreadPoolExecutor(workers) as ex:
        list(ex.map(work, range(0, n, chunk)))
    return out
