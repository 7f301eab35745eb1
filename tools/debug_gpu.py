"""Ad-hoc GPU parity probe: GPU hierarchy/solve vs the CPU oracle on golden cases."""
import sys, time, traceback
sys.path.insert(0, "/root/repo")
import numpy as np
from oracle import amg_oracle as O
from tests.cases import load, CASES
import paper_2602_23613_b200 as P

def cmp_csr(a, b):
    a = a.tocsr(); b = b.tocsr()
    same_pat = a.shape == b.shape and a.nnz == b.nnz and np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    if not same_pat:
        return f"PATTERN DIFF shape {a.shape} vs {b.shape} nnz {a.nnz} vs {b.nnz}"
    d = np.abs(a.data - b.data).max() / max(np.abs(b.data).max(), 1e-300) if a.nnz else 0.0
    return f"pattern ok, rel maxdiff {d:.2e}, bitexact {np.array_equal(a.data, b.data)}"

names = sys.argv[1:] or CASES
for name in names:
    print("=" * 20, name, flush=True)
    try:
        c = load(name)
        t = time.time()
        ho = O.hierarchy(c.system, c.meta["method"], meshes=c.meshes, rmaps=c.rmaps)
        to = time.time() - t
        t = time.time()
        hg = P.build_hierarchy(c.system, c.meta["method"], meshes=c.meshes, rmaps=c.rmaps)
        tg = time.time() - t
        print(f"setup oracle {to:.3f}s gpu {tg:.3f}s (device {hg.setup_seconds:.4f}s) depth {hg.depth}/{ho.depth} stalled {hg.stalled}/{ho.stalled} notes {hg.notes}/{ho.notes}")
        for ell in range(min(hg.depth, ho.depth)):
            lg, lo = hg.levels[ell], ho.levels[ell]
            print(f" L{ell} n {lg.n}/{lo.n} A: {cmp_csr(lg.A, lo.A)}")
            print(f"     G: {cmp_csr(lg.G, lo.G)}")
            if lo.P is not None and lg.P is not None:
                so, sg = lo.splitting, lg.splitting
                po = [(p.dof1, p.dof2, p.sign1, p.sign2, p.tail, p.mid, p.head) for p in so.pairs]
                pg = [tuple(p) for p in sg.pairs]
                print(f"     pairs {len(pg)}/{len(po)} equal {pg == po}; interior equal {np.array_equal(sg.interior_dofs, so.interior_dofs)}; cG equal {np.array_equal(sg.coarse_nodes, so.coarse_nodes) if so.coarse_nodes is not None else 'n/a'}")
                if pg != po:
                    for i, (a, b) in enumerate(zip(pg, po)):
                        if a != b:
                            print("     first pair diff", i, a, b); break
                print(f"     P: {cmp_csr(lg.P, lo.P)}")
                print(f"     l1 rel {np.abs(lg.l1.d - lo.l1).max() / lo.l1.max():.2e}; patches equal {all(np.array_equal(a, b) for a, b in zip(lg.patches.patches, lo.patches.patches)) and len(lg.patches.patches) == len(lo.patches.patches)}; waves {lg.patches.waves.max() + 1 if len(lg.patches.waves) else 0}")
        b = c.z["pcg_b"]
        vo = O.vcycle(ho, b); vg = P.vcycle(hg, b)
        print(f" vcycle rel diff {np.linalg.norm(vg - vo) / np.linalg.norm(vo):.2e}")
        xo, ro = O.pcg(c.system.A, b, precond=lambda r: O.vcycle(ho, r), tol=1e-8)
        t = time.time()
        xg, rg = P.pcg(c.system.A, b, precond=lambda r: P.vcycle(hg, r), tol=1e-8)
        print(f" pcg iters {rg.iterations}/{ro.iterations} conv {rg.converged} x rel diff {np.linalg.norm(xg - xo) / np.linalg.norm(xo):.2e} time {time.time() - t:.4f}s")
        print("   hist gpu", " ".join(f"{v:.3e}" for v in rg.residual_history))
        print("   hist ref", " ".join(f"{v:.3e}" for v in ro.residual_history))
        if "amg_x" in c.z:
            xa, ra = P.amg_solve(hg, c.z["amg_b"], x0=c.z["amg_x0"], tol=1e-8, maxit=200)
            print(f" amg iters {ra.iterations}/{c.meta['amg_iters']} rel diff {np.linalg.norm(xa - c.z['amg_x']) / np.linalg.norm(c.z['amg_x']):.2e} note '{ra.note}'")
    except Exception:
        traceback.print_exc()
