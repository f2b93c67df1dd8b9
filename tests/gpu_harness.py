"""Test-side glue between the fp64 oracle (NCHW, per-unit arrays) and the CUDA
library (NHWC, packed fp32).  Only layout conversion -- no PETRA arithmetic."""
import numpy as np

import synth
from oracle import models as OM
from oracle.units import DSUnit, RevUnit, StemUnit, TailUnit
from paper_2406_02052_b200 import models as PM
from paper_2406_02052_b200 import _lib as L


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def nhwc(x):
    return np.ascontiguousarray(np.asarray(x).transpose(0, 2, 3, 1)) if x.ndim == 4 else x


def nchw(x):
    return np.ascontiguousarray(np.asarray(x).transpose(0, 3, 1, 2))


def oracle_to_product_units(units):
    """Product unit list equivalent to an oracle unit list (same architecture)."""
    out = []
    for u in units:
        if isinstance(u, RevUnit):
            out.append(PM.Unit(L.UNIT_REV, u.dst, [(l.cin, l.cout, l.k, l.stride) for l in u.phi.layers]))
        elif isinstance(u, DSUnit):
            out.append(PM.Unit(L.UNIT_DS, u.dst, [(l.cin, l.cout, l.k, l.stride) for l in u.phi.layers],
                               [(p.cin, p.cout, p.k, p.stride) for p in (u.pa, u.pb)]))
        elif isinstance(u, StemUnit):
            l = u.layer
            out.append(PM.Unit(L.UNIT_STEM, 0, [(l.cin, l.cout, l.k, l.stride)], maxpool=int(u.maxpool)))
        elif isinstance(u, TailUnit):
            out.append(PM.Unit(L.UNIT_TAIL, classes=u.classes))
    return out


def pack_params(units):
    """Oracle parameters -> (theta, buffers) in the library's packed layout."""
    th, bf = [], []
    for u in units:
        for name, p, _ in u.params():
            if name == "w" and p.ndim == 4:
                th.append(p.transpose(0, 2, 3, 1).ravel())
            else:
                th.append(p.ravel())
        for _, b in u.buffers():
            bf.append(b.ravel())
    return (np.concatenate(th).astype(np.float32),
            np.concatenate(bf).astype(np.float32) if bf else np.zeros(0, np.float32))


def pack_like(units, arrays):
    """A list of per-parameter arrays (oracle order/layout) -> packed vector."""
    out, i = [], 0
    for u in units:
        for name, p, _ in u.params():
            a = arrays[i]
            out.append(a.transpose(0, 2, 3, 1).ravel() if (name == "w" and a.ndim == 4) else a.ravel())
            i += 1
    return np.concatenate(out)


def pack_buffers(units):
    return np.concatenate([b.ravel() for u in units for _, b in u.buffers()]) if any(
        True for u in units for _ in u.buffers()) else np.zeros(0)


def per_tensor_rel(units, got, want):
    """Relative error per parameter tensor (list of (name, rel))."""
    res, off = [], 0
    for ui, u in enumerate(units):
        for name, p, _ in u.params():
            n = p.size
            res.append((f"u{ui}.{name}", rel(got[off:off + n], want[off:off + n])))
            off += n
    return res


def rand_params(units, seed):
    OM.init_params(units, seed)
    i = 0
    for u in units:
        for name, p, _ in u.params():
            if name == "gamma":
                p[...] = 1.0 + 0.2 * synth.normal(p.shape, seed, 100, i)
            elif name in ("beta", "b"):
                p[...] = 0.1 * synth.normal(p.shape, seed, 101, i)
            i += 1
    return units


def elementwise(got, want):
    """Element-wise view of a comparison (per-tensor norms hide a wrong
    row): max |err| / max |want|, and the fraction of elements whose error exceeds
    1e-2 of the tensor's rms ("outliers")."""
    a, b = np.asarray(got, np.float64).ravel(), np.asarray(want, np.float64).ravel()
    err = np.abs(a - b)
    rms = np.sqrt(np.mean(b * b)) if b.size else 0.0
    mx = float(err.max() / max(np.abs(b).max(), 1e-30)) if b.size else 0.0
    out = float(np.mean(err > 1e-2 * max(rms, 1e-30))) if b.size else 0.0
    return mx, out
