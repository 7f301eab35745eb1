"""Generate the golden fixtures that pin the oracle to the reference itself.

Run in the build container only (needs /root/reference, which does not exist
on the GPU box):

    python tests/golden/make_golden.py

For every case it runs the UNMODIFIED reference (``hcurl_amg`` imported from
/root/reference/pkg/src) and stores its inputs and outputs in
``tests/golden/<case>.npz``.  Small cases keep full matrices; the config-1
case keeps sha256 digests of every array plus the small outputs (x, history,
A_c) so the fixture stays small.  Versions of numpy/scipy are recorded.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import scipy

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from hcurl_amg import fem, mesh as rmesh, multilevel, splitting, sparse  # noqa: E402

from paper_2602_23613_b200 import kuhn  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def put_csr(out, key, M):
    out[key + "_indptr"] = M.indptr.astype(np.int64)
    out[key + "_indices"] = M.indices.astype(np.int64)
    out[key + "_data"] = M.data
    out[key + "_shape"] = np.array(M.shape, dtype=np.int64)


def digest_csr(M):
    return {"shape": list(M.shape), "nnz": int(M.nnz),
            "pattern": sha(M.indptr.astype(np.int64), M.indices.astype(np.int64)),
            "values": sha(M.data)}


def run_case(name, system, method, meshes=None, rmaps=None, full=True, seed=0, amg=True):
    out = {}
    meta = {"case": name, "method": method, "numpy": np.__version__, "scipy": scipy.__version__}
    put_csr(out, "in_A", system.A)
    put_csr(out, "in_G", system.G)
    out["in_free_edges"] = np.asarray(system.free_edges, dtype=np.int64)
    if meshes is not None:
        out["chain_len"] = np.array([len(meshes)])
        for i, m in enumerate(meshes):
            out[f"mesh{i}_edges"] = np.asarray(m.edges, dtype=np.int64)
        for i, rm in enumerate(rmaps):
            out[f"rmap{i}_children"] = np.asarray(rm.coarse_edge_children, dtype=np.int64)
    h = multilevel.build_hierarchy(system, method, meshes=meshes, rmaps=rmaps)
    meta["depth"] = h.depth
    meta["stalled"] = bool(h.stalled)
    meta["notes"] = list(h.notes)
    meta["oc"] = multilevel.operator_complexity(h)
    meta["levels"] = []
    for ell, lv in enumerate(h.levels):
        d = {"n": int(lv.n), "A": digest_csr(lv.A), "G": digest_csr(lv.G)}
        if lv.P is not None:
            d["P"] = digest_csr(lv.P)
            sp_ = lv.splitting
            d["dump_sha"] = hashlib.sha256(splitting.dump_splitting(sp_).encode()).hexdigest()
            d["n_pairs"] = sp_.n_pairs
            d["n_interior"] = int(len(sp_.interior_dofs))
            d["n_patches"] = len(lv.patches.patches)
            d["l1"] = sha(lv.l1.d)
            out[f"L{ell}_pairs"] = np.array([tuple(p) for p in sp_.pairs], dtype=np.int64).reshape(-1, 7)
            out[f"L{ell}_interior"] = np.asarray(sp_.interior_dofs, dtype=np.int64)
            if sp_.coarse_nodes is not None:
                out[f"L{ell}_cG"] = np.asarray(sp_.coarse_nodes, dtype=np.int64)
            out[f"L{ell}_l1"] = lv.l1.d
            out[f"L{ell}_patch_sizes"] = np.array([len(p) for p in lv.patches.patches])
            out[f"L{ell}_patch_dofs"] = np.concatenate(lv.patches.patches).astype(np.int64)
            if full:
                put_csr(out, f"L{ell}_P", lv.P)
        if full or lv.n <= 400:
            put_csr(out, f"L{ell}_A", lv.A)
            put_csr(out, f"L{ell}_G", lv.G)
        meta["levels"].append(d)
    n = system.n
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, n)
    x, rep = multilevel.pcg(system.A, b, precond=lambda r: multilevel.vcycle(h, r), tol=1e-8)
    out["pcg_b"] = b
    out["pcg_x"] = x
    out["pcg_hist"] = rep.residual_history
    meta["pcg_iters"] = rep.iterations
    meta["pcg_converged"] = bool(rep.converged)
    out["vc_b"] = b
    out["vc_x"] = multilevel.vcycle(h, b)
    if amg:
        b2 = np.arange(1.0, n + 1.0)
        x0 = np.random.default_rng(seed + 1).uniform(-1, 1, n)
        xa, ra = multilevel.amg_solve(h, b2, x0=x0, tol=1e-8, maxit=200)
        out["amg_b"] = b2
        out["amg_x0"] = x0
        out["amg_x"] = xa
        out["amg_hist"] = ra.residual_history
        meta["amg_iters"] = ra.iterations
        meta["amg_converged"] = bool(ra.converged)
        meta["amg_note"] = ra.note
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "depth", h.depth, [lv.n for lv in h.levels], "pcg", rep.iterations,
          "size", os.path.getsize(os.path.join(HERE, f"{name}.npz")) // 1024, "KB")


def tri_chain(L, stripes=False, beta=0.01):
    meshes, rmaps = rmesh.refinement_chain(rmesh.uniform_tri_mesh(0), L)
    m = meshes[-1]
    mu = rmesh.assign_mu_stripes(m, L) if stripes else rmesh.uniform_mu(m)
    return meshes, rmaps, fem.assemble(m, mu, beta=beta)


def quad_chain(L, beta=0.01):
    meshes, rmaps = rmesh.refinement_chain(rmesh.uniform_quad_mesh(0), L)
    m = meshes[-1]
    return meshes, rmaps, fem.assemble(m, rmesh.uniform_mu(m), beta=beta)


def kats():
    """Known-answer tests taken from the reference's own unit tests."""
    out = {}
    # path graph of 5 nodes: C = [0, 2, 4] (tests/test_splitting.py:106-109)
    from hcurl_amg.splitting import classical_cf, augment_gradient
    pg = []
    for i in range(4):
        pg += [(i, i + 1, -1.0), (i + 1, i, -1.0)]
    pg += [(i, i, 2.0) for i in range(5)]
    r, c, v = zip(*pg)
    P5 = sparse.csr((v, (r, c)), shape=(5, 5))
    C, F = classical_cf(P5)
    out["path5_C"], out["path5_F"] = C, F
    aug = augment_gradient(sparse.csr(np.array([[1.0]])))
    out["aug1_G"] = aug.Gtilde.toarray()
    out["aug1_B"] = aug.boundary_cols
    # random symmetric graphs for C/F (tests/test_splitting.py:118-131)
    rng = np.random.default_rng(5)
    for t in range(5):
        M = rng.uniform(-1, 1, (30, 30)) * (rng.uniform(0, 1, (30, 30)) < 0.15)
        M = M + M.T + np.eye(30) * 5
        out[f"rand{t}_M"] = M
        C, F = classical_cf(sparse.csr(M))
        out[f"rand{t}_C"] = C
    np.savez_compressed(os.path.join(HERE, "kats.npz"), **out)


def api_inputs():
    """2D systems + nested mesh chains used by the ported reference API tests
    (tests/test_multilevel.py:25-30 tri_setup)."""
    out = {}
    for L, stripes in ((1, False), (2, False), (3, False), (3, True)):
        key = f"tri{L}{'s' if stripes else ''}"
        meshes, rmaps, s = tri_chain(L, stripes=stripes)
        put_csr(out, key + "_A", s.A)
        put_csr(out, key + "_G", s.G)
        out[key + "_free_edges"] = np.asarray(s.free_edges, dtype=np.int64)
        out[key + "_chain_len"] = np.array([len(meshes)])
        for i, m in enumerate(meshes):
            out[f"{key}_mesh{i}_edges"] = np.asarray(m.edges, dtype=np.int64)
        for i, rm in enumerate(rmaps):
            out[f"{key}_rmap{i}_children"] = np.asarray(rm.coarse_edge_children, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "api_inputs.npz"), **out)


def main():
    kats()
    api_inputs()
    meshes, rmaps, s = tri_chain(2)
    run_case("tri2_alg", s, "alg")
    meshes, rmaps, s = tri_chain(3, stripes=True)
    run_case("tri3s_alg", s, "alg")
    run_case("tri3s_ref", s, "ref", meshes, rmaps)
    meshes, rmaps, s = tri_chain(5, stripes=True)
    run_case("tri5s_alg", s, "alg")
    run_case("tri5s_ref", s, "ref", meshes, rmaps)
    meshes, rmaps, s = quad_chain(3)
    run_case("quad3_alg", s, "alg")
    run_case("quad3_ref", s, "ref", meshes, rmaps)
    run_case("kuhn4_c1", kuhn.config_system("c1", n=4), "alg")
    run_case("kuhn8_c2", kuhn.config_system("c2", n=8), "alg", full=False)
    run_case("kuhn8_c1", kuhn.config_system("c1"), "alg", full=False)


if __name__ == "__main__":
    main()
