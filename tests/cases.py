"""Shared loaders for the golden fixtures (tests/golden/*.npz) and seeded inputs."""

from __future__ import annotations

import hashlib
import json
import os
from types import SimpleNamespace

import numpy as np
import scipy.sparse as sp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["tri2_alg", "tri3s_alg", "tri3s_ref", "tri5s_alg", "tri5s_ref", "quad3_alg",
         "quad3_ref", "kuhn4_c1", "kuhn8_c2", "kuhn8_c1", "kuhn8_c3ref", "kuhn8_c2ref",
         "kuhn8_c4", "kuhn8_c5"]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def get_csr(z, key):
    shape = tuple(int(v) for v in z[key + "_shape"])
    M = sp.csr_matrix((z[key + "_data"], z[key + "_indices"].astype(np.int32),
                       z[key + "_indptr"].astype(np.int32)), shape=shape)
    return M


def digest_csr(M):
    return {"shape": list(M.shape), "nnz": int(M.nnz),
            "pattern": sha(M.indptr.astype(np.int64), M.indices.astype(np.int64)),
            "values": sha(M.data)}


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    meta = json.loads(str(z["meta"]))
    A, G = get_csr(z, "in_A"), get_csr(z, "in_G")
    system = SimpleNamespace(A=A, G=G, free_edges=z["in_free_edges"], n=A.shape[0])
    meshes = rmaps = None
    if "chain_len" in z:
        k = int(z["chain_len"][0])
        meshes = [SimpleNamespace(edges=z[f"mesh{i}_edges"], ne=len(z[f"mesh{i}_edges"]))
                  for i in range(k)]
        rmaps = [SimpleNamespace(coarse_edge_children=z[f"rmap{i}_children"]) for i in range(k - 1)]
    return SimpleNamespace(z=z, meta=meta, system=system, meshes=meshes, rmaps=rmaps)


def api_system(key):
    """(meshes, rmaps, system) of a 2D chain stored in golden/api_inputs.npz
    (the reference tests' tri_setup(L[, stripes]))."""
    z = np.load(os.path.join(GOLDEN, "api_inputs.npz"))
    A, G = get_csr(z, key + "_A"), get_csr(z, key + "_G")
    system = SimpleNamespace(A=A, G=G, free_edges=z[key + "_free_edges"], n=A.shape[0])
    k = int(z[key + "_chain_len"][0])
    meshes = [SimpleNamespace(edges=z[f"{key}_mesh{i}_edges"], ne=len(z[f"{key}_mesh{i}_edges"])) for i in range(k)]
    rmaps = [SimpleNamespace(coarse_edge_children=z[f"{key}_rmap{i}_children"]) for i in range(k - 1)]
    return meshes, rmaps, system


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
