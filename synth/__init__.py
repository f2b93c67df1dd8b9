"""Seeded synthetic inputs shared by the oracle tests and the GPU parity tests.

This module holds NONE of PETRA's arithmetic: it only draws random numbers.
Both sides (``oracle/`` and the CUDA path) receive the arrays it produces, so
parity tests compare the two implementations on identical inputs
(DESIGN.md "Input recipe").

Recipe (SURVEY.md §8(d) "Synthetic inputs"):
  * host draws use numpy ``PCG64(seed)``; micro-batch ``m`` of stream ``seed``
    uses ``PCG64([seed, m])`` so every micro-batch is reproducible on its own;
  * images are i.i.d. N(0, 1) per pixel (matches per-channel normalised data);
  * labels are uniform on [0, classes);
  * conv / linear weights are Kaiming-uniform U(+-sqrt(6 / fan_in)), BN gamma=1,
    beta=0, biases 0, running mean 0 / var 1, momentum buffers 0
    (SURVEY.md §8(c) reading c17 -- the paper does not state its init).
"""
from __future__ import annotations

import numpy as np

__all__ = ["rng", "images", "labels", "kaiming_uniform", "normal", "class_gaussian_batch"]


def rng(seed: int, *stream: int) -> np.random.Generator:
    """Counter-style generator: one independent stream per (seed, *stream)."""
    return np.random.Generator(np.random.PCG64([int(seed), *[int(s) for s in stream]]))


def images(shape, seed: int = 0, mb: int = 0) -> np.ndarray:
    """N(0,1) float64 array of ``shape`` for micro-batch ``mb``."""
    return rng(seed, 1, mb).standard_normal(tuple(shape))


def normal(shape, seed: int, *stream: int, scale: float = 1.0) -> np.ndarray:
    return scale * rng(seed, 2, *stream).standard_normal(tuple(shape))


def labels(batch: int, classes: int, seed: int = 0, mb: int = 0) -> np.ndarray:
    """Uniform int64 labels in [0, classes)."""
    return rng(seed, 3, mb).integers(0, classes, size=int(batch), dtype=np.int64)


def kaiming_uniform(shape, fan_in: int, seed: int, index: int) -> np.ndarray:
    """U(-b, b) with b = sqrt(6 / fan_in) -- tensor ``index`` of parameter seed ``seed``."""
    b = float(np.sqrt(6.0 / fan_in))
    return rng(seed, 4, index).uniform(-b, b, size=tuple(shape))


def class_gaussian_batch(shape, classes: int, seed: int, mb: int, sep: float = 2.0):
    """Class-conditional Gaussian images (SPEC.md:584 idea): learnable synthetic data.

    Returns (x, y). Class means are fixed random directions scaled by ``sep``.
    """
    g = rng(seed, 5, mb)
    y = g.integers(0, classes, size=shape[0], dtype=np.int64)
    means = rng(seed, 6).standard_normal((classes,) + tuple(shape[1:]))
    means *= sep / np.sqrt(np.prod(shape[1:]))
    x = g.standard_normal(tuple(shape)) + means[y] * np.sqrt(np.prod(shape[1:]))
    return x, y
