"""Generate the golden fixtures that pin the oracle (and, through it, the GPU
path) to the reference implementation.

Runs ONLY in the build container, where the reference package is mounted at
/root/reference (read-only).  It imports `terngemm` from there, builds formats
and runs every in-scope reference kernel on seeded integer- and real-valued
inputs, and writes compact .npz files next to this script:

  formats.npz  W -> Tcsc / BlockedTcsc / InterleavedBlockedTcsc(+symmetric) /
               SymmetricInterleavedTcsc / CompressedTcsc arrays, for many
               shapes, block sizes and group sizes
  kernels.npz  X, b and the reference kernels' fp32 outputs (+ OpCounts) for
               base / unrolled / blocked / interleaved_blocked /
               vectorized_optimal / compressed / vertical / horizontal, plus
               oracle_gemm, on integer AND real X
  cfg1.npz     the BASELINE cfg1 workload (seed 1, SURVEY.md 8(d) recipe):
               reference Tcsc arrays and gemm_base output

Usage:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
Nothing in the GPU tests, smoke() or bench.py reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import terngemm as tg  # noqa: E402  (the reference)

from paper_2510_06957_b200.workloads import make_inputs  # noqa: E402


def rand_w(rng, K, N, kind):
    if kind == "unstructured":
        return rng.integers(-1, 2, size=(K, N)).astype(np.int8)
    if kind == "sparse":
        u = rng.random((K, N))
        return np.where(u < 0.1, 1, np.where(u < 0.17, -1, 0)).astype(np.int8)
    if kind == "lopsided":  # many more +1 than -1: long remainders, many dummies
        u = rng.random((K, N))
        return np.where(u < 0.45, 1, np.where(u < 0.5, -1, 0)).astype(np.int8)
    if kind == "zero":
        return np.zeros((K, N), np.int8)
    if kind == "dense":
        return np.where(rng.random((K, N)) < 0.5, 1, -1).astype(np.int8)
    raise ValueError(kind)


def put_fmt(store, key, fmt):
    for name in ("col_start_pos", "row_index_pos", "col_start_neg", "row_index_neg", "all_indices", "col_segment_ptr",
                 "indices", "col_ptr", "codes"):
        if hasattr(fmt, name):
            store[f"{key}.{name}"] = np.asarray(getattr(fmt, name))


def formats_fixture():
    rng = np.random.default_rng(20251007)
    store, index = {}, []
    shapes = [(1, 1), (1, 4), (4, 2), (2, 8), (5, 3), (7, 12), (13, 8), (33, 5), (64, 16), (100, 20), (257, 12), (300, 40)]
    kinds = ["unstructured", "sparse", "lopsided", "zero", "dense"]
    cid = 0
    # worked example (conftest.py:24-29) and the SURVEY 8x4 symmetric example
    ws = [np.array([[1, 0], [0, -1], [-1, 0], [1, 0]], np.int8)]
    w8 = np.zeros((8, 4), np.int8)
    w8[0:2, 0] = 1
    w8[2:4, 0] = -1
    w8[5, 1] = 1
    ws.append(w8)
    for (K, N) in shapes:
        for kind in kinds:
            if kind in ("zero", "dense") and K * N > 2000:
                continue
            ws.append(rand_w(rng, K, N, kind))
    for W in ws:
        K, N = W.shape
        key = f"c{cid}"
        store[f"{key}.W"] = W
        entry = {"key": key, "K": K, "N": N, "formats": []}
        Wt = tg.TernaryDense(W)
        put_fmt(store, f"{key}.tcsc", tg.tcsc_from_dense(Wt))
        entry["formats"].append({"name": "tcsc"})
        big = K * N > 2000
        bset = {None, 7, 64} if big else {None, 1, 2, 3, 7, 16, 64, K}
        for B in sorted(bset, key=lambda x: -1 if x is None else x):
            if B is not None and B > K + 1:
                continue
            f = tg.blocked_from_dense(Wt, B)
            name = f"blocked_B{B}"
            put_fmt(store, f"{key}.{name}", f)
            entry["formats"].append({"name": name, "B": B, "resolved_B": f.B})
            for g in ((1, 2, 3) if big else (1, 2, 3, 4)):
                for sym in (False, True):
                    if sym and N % 4:
                        continue
                    f2 = tg.interleaved_blocked_from_dense(Wt, B, g, sym)
                    name2 = f"ib_B{B}_g{g}_s{int(sym)}"
                    put_fmt(store, f"{key}.{name2}", f2)
                    entry["formats"].append({"name": name2, "B": B, "g": g, "sym": sym, "resolved_B": f2.B,
                                             "nnz": f2.nnz, "bytes": f2.format_bytes()})
        # SymmetricInterleavedTcsc (variants.py:540-631) and CompressedTcsc (variants.py:451-532)
        if N % 4 == 0:
            for g in (1, 2, 3, 4):
                f3 = tg.symmetric_from_dense(Wt, g)
                put_fmt(store, f"{key}.sym_g{g}", f3)
                entry["formats"].append({"name": f"sym_g{g}", "g": g, "nnz": f3.nnz, "dummies": f3.dummy_count,
                                         "bytes": f3.format_bytes()})
        fc = tg.compressed_from_dense(Wt)
        put_fmt(store, f"{key}.compressed", fc)
        entry["formats"].append({"name": "compressed", "nnz": fc.nnz, "bytes": fc.format_bytes()})
        index.append(entry)
        cid += 1
    store["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "formats.npz"), **store)
    print("formats.npz:", cid, "matrices")


def kernels_fixture():
    rng = np.random.default_rng(6957)
    store, index = {}, []
    cases = [(1, 1, 4), (1, 4, 4), (2, 8, 4), (3, 5, 8), (4, 16, 4), (5, 17, 8), (7, 33, 12), (9, 64, 16),
             (4, 100, 20), (6, 130, 8), (8, 257, 12), (5, 300, 40), (12, 80, 24)]
    cid = 0
    for (M, K, N) in cases:
        for kind in ("unstructured", "sparse", "lopsided"):
            for xmode in ("int", "uniform", "normal"):
                W = rand_w(rng, K, N, kind)
                if xmode == "int":
                    X = rng.integers(-8, 9, (M, K)).astype(np.float32)
                    b = rng.integers(-8, 9, N).astype(np.float32)
                elif xmode == "uniform":
                    X = (rng.random((M, K)) * 2 - 1).astype(np.float32)
                    b = rng.standard_normal(N).astype(np.float32)
                else:
                    X = rng.standard_normal((M, K)).astype(np.float32)
                    b = rng.standard_normal(N).astype(np.float32)
                key = f"k{cid}"
                Wt, Xt, bt = tg.TernaryDense(W), tg.DenseMatrix(X), tg.BiasVector(b)
                store[f"{key}.W"], store[f"{key}.X"], store[f"{key}.b"] = W, X, b
                runs = []

                def rec(name, pair, **meta):
                    y, ops = pair
                    store[f"{key}.{name}"] = y.values
                    runs.append({"name": name, "adds": int(ops.adds), "mults": int(ops.mults), **meta})

                t = tg.tcsc_from_dense(Wt)
                rec("base", tg.gemm_base(Xt, t, bt, counted=True))
                for uf, mr, nr in ((12, 4, 4), (3, 2, 1), (1, 1, 2), (5, 4, 2)):
                    cfg = tg.GemmConfig(uf=uf, mr=mr, nr=nr)
                    rec(f"unrolled_u{uf}_m{mr}_n{nr}", tg.gemm_unrolled(Xt, t, bt, cfg, counted=True), uf=uf, mr=mr, nr=nr)
                for B, uf, mr in ((None, 12, 4), (7, 5, 2), (3, 1, 4), (16, 4, 1)):
                    cfg = tg.GemmConfig(uf=uf, mr=mr, b=B)
                    f = tg.blocked_from_dense(Wt, B)
                    rec(f"blocked_B{B}_u{uf}_m{mr}", tg.gemm_blocked(Xt, f, bt, cfg, counted=True), B=B, uf=uf, mr=mr)
                for B, g, mr in ((None, 2, 4), (5, 3, 2), (16, 1, 1), (3, 4, 4)):
                    cfg = tg.GemmConfig(mr=mr, b=B, g=g)
                    f = tg.interleaved_blocked_from_dense(Wt, B, g)
                    rec(f"ib_B{B}_g{g}_m{mr}", tg.gemm_interleaved_blocked(Xt, f, bt, cfg, counted=True), B=B, g=g, mr=mr)
                if N % 4 == 0:
                    Xp = tg.pad_input(Xt)
                    for B, g in ((None, 2), (7, 1), (16, 3)):
                        f = tg.interleaved_blocked_from_dense(Wt, B, g, symmetric_cols=True)
                        for alpha in (None, 0.25, 0.1):
                            rec(f"opt_B{B}_g{g}_a{alpha}",
                                tg.gemm_vectorized_optimal(Xp, f, bt, alpha, counted=True), B=B, g=g, alpha=alpha,
                                n_indices=int(f.all_indices.shape[0]), nb=f.num_blocks)
                rec("compressed", tg.gemm_compressed(Xt, tg.compressed_from_dense(Wt), bt, counted=True))
                if N % 4 == 0:
                    Xp = tg.pad_input(Xt)
                    for g in (2, 1, 3):
                        f = tg.symmetric_from_dense(Wt, g)
                        for alpha in (None, 0.25):
                            rec(f"vertical_g{g}_a{alpha}", tg.gemm_vertical(Xp, f, bt, alpha, counted=True), g=g,
                                alpha=alpha, n_indices=int(f.indices.shape[0]))
                            rec(f"horizontal_g{g}_a{alpha}", tg.gemm_horizontal(Xp, f, bt, alpha, counted=True), g=g,
                                alpha=alpha, n_indices=int(f.indices.shape[0]))
                for alpha in (None, 0.25):
                    store[f"{key}.oracle_a{alpha}"] = tg.oracle_gemm(Xt, Wt, bt, alpha).values
                index.append({"key": key, "M": M, "K": K, "N": N, "wkind": kind, "xmode": xmode,
                              "nnz": int(np.count_nonzero(W)), "runs": runs})
                cid += 1
    store["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **store)
    print("kernels.npz:", cid, "cases")


def cfg1_fixture():
    W, X, b = make_inputs("cfg1")
    t = tg.tcsc_from_dense(tg.TernaryDense(W))
    y = tg.gemm_base(tg.DenseMatrix(X), t, tg.BiasVector(b))
    store = {
        "col_start_pos": t.col_start_pos, "col_start_neg": t.col_start_neg,
        "row_index_pos": t.row_index_pos, "row_index_neg": t.row_index_neg,
        "Y_base": y.values,
        "oracle": tg.oracle_gemm(tg.DenseMatrix(X), tg.TernaryDense(W), tg.BiasVector(b)).values,
    }
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **store)
    print("cfg1.npz: nnz", t.nnz)


def files_fixture():
    """TGW1 / TGS1 bytes written by the reference (io.py) and its seeded generators."""
    import io as _io

    from terngemm import io as tio

    def dump(fn, obj):
        fh = _io.BytesIO()
        fn(obj, fh)
        return np.frombuffer(fh.getvalue(), dtype=np.uint8)

    store = {}
    meta = []
    for i, (K, N, s, seed) in enumerate([(24, 8, "1/2", 6), (37, 12, "1/4", 1), (130, 20, "3/5", 2), (9, 4, "1", 3)]):
        w = tg.gen_ternary(K, N, s, seed)
        store[f"f{i}_W"] = w.values
        store[f"f{i}_dense"] = dump(tio.save_dense, w)
        fmts = {
            "tcsc": tg.tcsc_from_dense(w),
            "blocked": tg.blocked_from_dense(w, B=8),
            "interleaved_blocked": tg.interleaved_blocked_from_dense(w, B=8, g=2),
            "compressed": tg.compressed_from_dense(w),
        }
        if N % 4 == 0:
            fmts["interleaved_blocked_sym"] = tg.interleaved_blocked_from_dense(w, B=8, g=2, symmetric_cols=True)
            fmts["symmetric"] = tg.symmetric_from_dense(w, g=2)
        for name, fmt in fmts.items():
            store[f"f{i}_{name}"] = dump(tio.save_sparse, fmt)
        store[f"f{i}_interleaved"] = dump(tio.save_sparse, tg.interleaved_from_dense(w, g=2))  # not supported here
        meta.append({"K": K, "N": N, "s": s, "seed": seed, "formats": sorted(fmts)})
        store[f"f{i}_gen_input"] = tg.gen_input(5, K, seed + 1).values
        store[f"f{i}_gen_bias"] = tg.gen_bias(N, seed + 2).values
        store[f"f{i}_gen_uniform"] = tg.gen_input_uniform(3, K, seed).values
    store["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "files.npz"), **store)
    print("files.npz:", len(meta), "matrices")


if __name__ == "__main__":
    files_fixture()
    formats_fixture()
    kernels_fixture()
    cfg1_fixture()
