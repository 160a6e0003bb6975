"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This module holds NONE of the method's arithmetic: it only loads the parameter
sets (configs/*.json, plain data) and draws the plaintext-side random inputs
(messages, LUT entries, Shift amounts, RLWE message polynomials) from numpy's
Philox generator.  Encryption, scaling by Delta, SetupPolynomial etc. are done
independently by each side.  Recipe:
  messages  m ~ U(Z_t)
  LUT       f ~ U(Z_t)^t, t' = t
  Shift     message coefficients ~ U(Z_Q)^N, d ~ U[1, N-1]
"""
import json
import os

import numpy as np

_CFG_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs")


def load_config(name: str) -> dict:
    with open(os.path.join(_CFG_DIR, name + ".json")) as f:
        return json.load(f)


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[int(seed), int(stream)]))


def messages(cfg: dict, count: int, seed=None) -> np.ndarray:
    seed = cfg["seeds"]["msgs"] if seed is None else seed
    return _rng(seed, 1).integers(0, cfg["t"], size=count, dtype=np.uint64)


def lut(cfg: dict, seed=None, t=None) -> np.ndarray:
    seed = cfg["seeds"]["lut"] if seed is None else seed
    t = cfg["t"] if t is None else t
    return _rng(seed, 2).integers(0, t, size=t, dtype=np.uint64)


def rlwe_messages(cfg: dict, count: int, seed=None) -> np.ndarray:
    seed = cfg["seeds"]["msgs"] if seed is None else seed
    return _rng(seed, 3).integers(0, cfg["Q"], size=(count, cfg["N"]), dtype=np.uint64)


def shift_amounts(cfg: dict, count: int, seed=None) -> np.ndarray:
    seed = cfg["seeds"]["msgs"] if seed is None else seed
    return _rng(seed, 4).integers(1, cfg["N"], size=count, dtype=np.uint32)
