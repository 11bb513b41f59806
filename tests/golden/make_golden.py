"""tests/golden/make_golden.py — regenerate the golden fixtures from the
COMPILED REFERENCE (oracle/_ref, built from /root/reference/proj/src).

Run here (the reference only exists in this container):
    python tests/golden/make_golden.py
Writes tests/golden/*.npz. Each fixture stores the inputs, the reference
outputs, and the reference's pair counts / counters, so the GPU tests on the box
(where /root/reference does not exist) compare against the reference itself.
Cases follow the reference's own pinned tests (file:line in each entry).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)
    print("wrote", name, {k: np.asarray(v).shape for k, v in arrays.items()})


def truncated_case(name, dim, n, K, hk, d0, seed, src):
    u = O.ref_random_vector(n ** dim, seed)
    fast, cnt, _ = O.ref_truncated_fast(dim, n, K, hk, d0, u)
    leaf, pairs = O.ref_truncated_dense(dim, n, K, hk, d0, u, O.LEAF, O.MASS)
    point, ppairs = O.ref_truncated_dense(dim, n, K, hk, d0, u, O.POINT, O.MASS)
    pdiff, _ = O.ref_truncated_dense(dim, n, K, hk, d0, u, O.POINT, O.DIFFERENCE)
    save(name, dim=dim, n=n, K=K, horizon_kind=hk, delta0=d0, seed=seed, u=u, fast=fast,
         counters=cnt, dense_leaf=leaf, leaf_pairs=pairs, dense_point=point,
         point_pairs=ppairs, dense_point_diff=pdiff, src=src)


def main():
    O.build(ref=True)
    # test_operators.cpp:55-87 — fast == dense Leaf (the reference's own pins)
    truncated_case("trunc_2d_n64_k0", 2, 64, 0, 0, 0.5, 42, "test_operators.cpp:56-65")
    truncated_case("trunc_1d_n2048_k3_bump", 1, 2048, 3, 1, 0.25, 43, "test_operators.cpp:66-76")
    truncated_case("trunc_3d_n8_k0", 3, 8, 0, 0, 0.5, 44, "test_operators.cpp:77-86")
    # test_operators.cpp:89-104 linearity case grid (K=2 bump n=512) and the
    # cfg0 grid (n=4096, delta=0.02) for K=0..3 — the conditioning probe
    truncated_case("trunc_1d_n512_k2_bump", 1, 512, 2, 1, 0.25, 1, "test_operators.cpp:89-104")
    for K in range(4):
        truncated_case(f"trunc_1d_n4096_k{K}_d002", 1, 4096, K, 0, 0.02, 1, "SURVEY.md §6 cfg0 grid")
    truncated_case("trunc_2d_n128_k0_bump", 2, 128, 0, 1, 0.05, 5, "2D bump, K=0")

    # kernel algebra: test_kernel.cpp:78-140
    polys = {f"p{K}": O.ref_match_polynomial(K) for K in range(5)}
    splits = {}
    for K in range(4):
        p, t = O.ref_split(K)
        splits[f"split_poly{K}"] = p
        splits[f"split_tail{K}"] = t
    s = (np.arange(2000) + 0.5) / 2000.0
    kap = {f"kappa{K}": O.ref_kappa(K, s) for K in range(4)}
    save("kernel_algebra", s=s, **polys, **splits, **kap)

    # smooth / full / split: test_operators.cpp:136-195 (1D n=256, delta=1/4)
    n = 256
    u = O.ref_random_vector(n, 17)
    smooth, sp = O.ref_smooth_dense(1, n, 2, 0, 0.25, u)
    full, fp = O.ref_full_dense(1, n, 0, 0, 0, 0.25, u)
    sp_pd = O.ref_apply_split(1, n, 2, 0, 0.25, u, truncated=1)
    sp_fl = O.ref_apply_split(1, n, 2, 0, 0.25, u, truncated=0)
    ones = np.ones(n)
    sp_ones = O.ref_apply_split(1, n, 1, 0, 0.25, ones, truncated=0)
    save("split_1d_n256", u=u, smooth_k2=smooth, smooth_pairs=sp, full=full, full_pairs=fp,
         split_k2_pointdiff=sp_pd, split_k2_fastleafmass=sp_fl, split_k1_ones=sp_ones,
         src="test_operators.cpp:136-195")
    # full dense families with a bump horizon, 1D and 2D (test_operators.cpp:235-246)
    out = {}
    for dim, n in ((1, 256), (2, 16)):
        u = O.ref_random_vector(n ** dim, 11)
        out[f"u{dim}"] = u
        for fam in range(4):
            for div in (0, 1):
                r, p = O.ref_full_dense(dim, n, fam, 2, 1, 0.25, u, divergence=div)
                out[f"full{dim}_f{fam}_div{div}"] = r
                out[f"pairs{dim}_f{fam}_div{div}"] = p
    save("full_families", **out)

    # BASELINE-kernel direct sums through coefficient_fn:
    # fractional |r|^-alpha, per-node delta(x), C(x) and (kappa_x+kappa_y)/2.
    rng = np.random.default_rng(1905)
    cases = {}
    for tag, dim, n, alpha, lo, hi in (("1d", 1, 2048, 1.8, 5, 40), ("2d", 2, 64, 3.0, 4, 12),
                                       ("3d", 3, 16, 3.5, 2, 4)):
        N = n ** dim
        h = 1.0 / n
        u = O.ref_random_vector(N, 21)
        delta = h * (lo + (hi - lo) * rng.random(N))
        cx = 0.5 + rng.random(N)
        kappa = np.exp(0.5 * rng.standard_normal(N))
        r1, p1 = O.ref_full_dense_general(dim, n, delta, cx, kappa, alpha, u)
        r0, p0 = O.ref_full_dense_general(dim, n, delta, None, None, alpha, u)
        cases.update({f"{tag}_u": u, f"{tag}_delta": delta, f"{tag}_cx": cx, f"{tag}_kappa": kappa,
                      f"{tag}_alpha": alpha, f"{tag}_kw": r1, f"{tag}_kw_pairs": p1,
                      f"{tag}_plain": r0, f"{tag}_plain_pairs": p0})
    # cfg0 operator (clip flavour the reference can express): n=4096, delta=0.02, s=0.25
    n = 4096
    u = O.ref_random_vector(n, 1)
    delta = np.full(n, 0.02)
    cd = 0.75 / 0.02 ** 1.5
    r, p = O.ref_full_dense_general(1, n, delta, np.full(n, cd), None, 1.5, u)
    cases.update(cfg0_u=u, cfg0_out_clip=r, cfg0_pairs=p, cfg0_cdelta=cd)
    save("fractional_general", **cases)

    # Krylov consumer (test_solve.cpp:73-159): manufactured solution
    # u* = sin(2 pi x) x (1 - x), f = -L u* via the dense Leaf apply
    sol = {}
    for tag, n, hk, tol in (("cg_n512", 512, 0, 1e-10), ("cgnr_n256_bump", 256, 1, 1e-10),
                            ("cg_n128_2it", 128, 0, 1e-14)):
        x = (np.arange(n) + 0.5) / n
        ustar = np.sin(2 * np.pi * x) * x * (1 - x)
        L, _ = O.ref_truncated_dense(1, n, 0, hk, 0.25, ustar, O.LEAF, O.MASS)
        f = -L
        max_iter = 2 if tag == "cg_n128_2it" else 10 * n
        u, it, res, conv, m = O.ref_solve_truncated(1, n, 0, hk, 0.25, f, tol, max_iter)
        sol.update({f"{tag}_ustar": ustar, f"{tag}_f": f, f"{tag}_u": u, f"{tag}_iters": it,
                    f"{tag}_residual": res, f"{tag}_converged": conv, f"{tag}_method": m,
                    f"{tag}_tol": tol, f"{tag}_max_iter": max_iter})
        if tag != "cg_n128_2it":
            a = -O.ref_assemble_dense(1, n, 3, 0, hk, 0.25)
            sol[f"{tag}_direct"] = O.ref_dense_direct_solve(a, f)
    # dense CG (the "dense matvec" subcase)
    n = 512
    u, it, res, conv, m = O.ref_solve_truncated(1, n, 0, 0, 0.25, sol["cg_n512_f"], 1e-10, 10 * n, use_dense=True)
    sol.update(cg_n512_dense_u=u, cg_n512_dense_iters=it, cg_n512_dense_residual=res)
    save("solve_dirichlet", src="test_solve.cpp:73-159, nonloc_main.cpp:189-222", **sol)

    # assemble_dense_matrix (operators.cpp:262-303): truncated K=1 constant
    # (test_solve.cpp:60-71 symmetry case), K=0 bump Leaf/Point x Mass/Difference,
    # full InverseS bump, 2-D K=0
    asm = {}
    for tag, dim, n, fam, K, hk, d0, rule, form, div in (
            ("k1_const_leaf_mass", 1, 128, 3, 1, 0, 0.25, O.LEAF, O.MASS, 0),
            ("k0_bump_leaf_mass", 1, 128, 3, 0, 1, 0.25, O.LEAF, O.MASS, 0),
            ("k0_bump_point_diff", 1, 128, 3, 0, 1, 0.25, O.POINT, O.DIFFERENCE, 0),
            ("inverse_s_bump", 1, 128, 0, 0, 1, 0.25, O.POINT, O.DIFFERENCE, 0),
            ("inverse_s_bump_div", 1, 128, 0, 0, 1, 0.25, O.POINT, O.DIFFERENCE, 1),
            ("k0_2d_leaf_mass", 2, 16, 3, 0, 1, 0.25, O.LEAF, O.MASS, 0)):
        asm[tag] = O.ref_assemble_dense(dim, n, fam, K, hk, d0, rule, form, divergence=div)
    save("assemble_dense", src="operators.cpp:262-303", **asm)

    # Step-1 tree API (tree.hpp:31-53; test_tree.cpp:83-133, 214-249):
    # decompose_region panel lists, count_recur_calls, accumulate_moments
    rng = np.random.default_rng(77)
    tr = {}
    k = 0
    for dim, n in ((1, 64), (1, 1024), (2, 32), (3, 8)):
        for _ in range(6):
            c = rng.random(dim)
            r = 0.02 + 0.5 * rng.random()
            lv, ix, rc = O.ref_decompose(dim, n, c, r)
            tr.update({f"d{k}_dim": dim, f"d{k}_n": n, f"d{k}_c": c, f"d{k}_r": r, f"d{k}_levels": lv,
                       f"d{k}_indices": ix, f"d{k}_recur": rc})
            k += 1
    tr["ndecomp"] = k
    for dim, n in ((1, 256), (2, 32), (3, 8)):
        radii = 0.05 + 0.3 * rng.random(n ** dim)
        tr[f"radii{dim}"] = radii
        tr[f"recur{dim}"] = O.ref_count_recur_calls(dim, n, radii)
    for dim, n, K in ((1, 16, 0), (1, 16, 3), (2, 8, 0), (3, 4, 0)):
        u = O.ref_random_vector(n ** dim, 9)
        m, adds = O.ref_moments(dim, n, K, u)
        tr[f"mom{dim}_{K}_u"] = u
        tr[f"mom{dim}_{K}"] = m
        tr[f"mom{dim}_{K}_adds"] = adds
    save("tree_api", src="tree.hpp:31-53, tree.cpp", **tr)


if __name__ == "__main__":
    main()
