"""Helpers to unpack the committed golden fixtures (tests/golden/*.npz)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def corpus_cases():
    """Yield dicts of the criterion-1-style corpus (gen_golden.gen_hseg_corpus)."""
    z = load("hseg_corpus.npz")
    meta = z["meta"]
    so = mo = ao = 0
    for row in meta:
        edge, bands, conn, weight, target, conv, nrec = row
        edge, bands, conn, target, conv, nrec = int(edge), int(bands), int(conn), int(target), int(conv), int(nrec)
        npx = edge * edge
        samples = z["samples"][so : so + bands * npx].reshape(bands, edge, edge)
        so += bands * npx
        recs = (
            z["merge_surv"][mo : mo + nrec],
            z["merge_abs"][mo : mo + nrec],
            z["merge_d"][mo : mo + nrec],
            z["merge_kind"][mo : mo + nrec],
        )
        mo += nrec
        assign = z["assign"][ao : ao + npx]
        ao += npx
        yield dict(edge=edge, bands=bands, conn=conn, weight=float(weight), target=target,
                   converged=bool(conv), records=recs, assign=assign, samples=samples)


LOG_KEYS = ("log_level", "log_row", "log_col", "log_survivor", "log_absorbed", "log_dissim", "log_kind")


def small_rhseg_cases():
    z = load("rhseg_small.npz")
    so = lo = lb = 0
    for row in z["meta"]:
        edge, bands, levels, w, tgt, st, conv, nrec = row
        edge, bands, levels, tgt, st, conv, nrec = map(int, (edge, bands, levels, tgt, st, conv, nrec))
        npx = edge * edge
        samples = z["samples"][so : so + bands * npx].reshape(bands, edge, edge)
        so += bands * npx
        labels = z["labels"][lb : lb + npx].reshape(edge, edge)
        lb += npx
        log = {k: z[k][lo : lo + nrec] for k in LOG_KEYS}
        lo += nrec
        yield dict(edge=edge, bands=bands, levels=levels, weight=float(w), target=tgt,
                   section_target=st, converged=bool(conv), samples=samples, labels=labels, log=log)


def scan_table_cases():
    z = load("scan_tables.npz")
    co = so = po = io = 0
    for n, nb, nnz in z["meta"]:
        n, nb, nnz = int(n), int(nb), int(nnz)
        yield dict(
            n=n, nb=nb,
            counts=z["counts"][co : co + n],
            sums=z["sums"][so : so + n * nb].reshape(n, nb),
            indptr=z["indptr"][po : po + n + 1],
            indices=z["indices"][io : io + nnz],
            adj_d=z["adj_d"][co : co + n], adj_j=z["adj_j"][co : co + n],
            non_d=z["non_d"][co : co + n], non_j=z["non_j"][co : co + n],
        )
        co += n
        so += n * nb
        po += n + 1
        io += nnz
