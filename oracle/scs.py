"""O0: the literal Soft Cosine Similarity of PAPER.md Eq. 11 (§IV-B).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Follows the paper's words
step by step on token embedding matrices, in fp64:

  "normalizing and concatenating their token embedding matrices, then multiplying
   by the transpose to yield a symmetric token similarity matrix C"
  "two alignment vectors V1 and V2 ... mark token ownership per prompt via binary
   indicators"
  SCS = V1^T C V2 / (sqrt(V1^T C V1) * sqrt(V2^T C V2) + sigma)   (Eq. 11)

"Normalizing" is read as per-row L2 normalisation (reading R2).
"""
from __future__ import annotations

import numpy as np


def normalize_rows(tokens: np.ndarray) -> np.ndarray:
    """Each token embedding row divided by its L2 norm (reading R2)."""
    t = np.asarray(tokens, dtype=np.float64)
    return t / np.sqrt((t * t).sum(axis=1, keepdims=True))


def scs_gram(tokens1: np.ndarray, tokens2: np.ndarray, sigma: float = 1e-6) -> float:
    """Eq. 11 literally: Gram matrix of the concatenated normalised rows, ownership vectors."""
    a = normalize_rows(tokens1)
    b = normalize_rows(tokens2)
    x = np.concatenate([a, b], axis=0)          # concatenated token matrix
    c = x @ x.T                                  # symmetric token similarity matrix C
    n1, n2 = a.shape[0], b.shape[0]
    v1 = np.concatenate([np.ones(n1), np.zeros(n2)])[:, None]   # column vectors
    v2 = np.concatenate([np.zeros(n1), np.ones(n2)])[:, None]
    num = (v1.T @ c @ v2).item()
    den = np.sqrt((v1.T @ c @ v1).item()) * np.sqrt((v2.T @ c @ v2).item()) + sigma
    return num / den


def prompt_vector(tokens: np.ndarray) -> np.ndarray:
    """The reduced prompt embedding a = V1^T X = sum of normalised token rows."""
    return normalize_rows(tokens).sum(axis=0)
