"""Regenerate the committed golden fixtures under tests/golden/.

  python tests/golden/make_golden.py

Two kinds of fixture:
  * ref_derive_seed.json — output of the REFERENCE's own seed derivation
    (proj/src/rng.hpp:10-25) compiled by oracle/build_ref.sh into
    oracle/_ref/ref_rng. Needs /root/reference (build container only).
  * oracle_*.json — vectors produced once by the CPU oracle (oracle/omc_oracle.c)
    and frozen: they pin the oracle against
    accidental change; the transport arithmetic itself is "parity unpinned"
    against the reference, which ships no transport code.
Large vectors are stored as sha256 digests of the raw little-endian arrays
plus a short explicit prefix.
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

PAIRS = 10_000


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def hexbits(x: float) -> str:
    return f"{np.float64(x).view(np.uint64):016x}"


def lookup_inputs(kind: int, n_nuc: int, seed: int):
    """The (nuclide, material, E) inputs of the lookup vectors (numpy PCG64, stable)."""
    rng = np.random.default_rng(seed)
    E = np.exp(rng.uniform(np.log(1e-6), np.log(3e7), PAIRS))
    E[:4] = [1e-5, 2e7, 1e-7, 5e7]
    nuc = rng.integers(0, n_nuc, PAIRS).astype(np.int32)
    mat = rng.integers(0, 3, PAIRS).astype(np.int32)
    return nuc, mat, E


def lookup_vectors(kind: int, bins: int):
    p = O.Problem(kind, 1234, bins)
    nuc, mat, E = lookup_inputs(kind, p.info.n_nuclides, 1000 + kind)
    idx = np.empty(PAIRS, np.int32)
    micro = np.empty((PAIRS, 4), np.float64)
    macro = np.empty((PAIRS, 4), np.float64)
    binv = np.empty(PAIRS, np.int32)
    for k in range(PAIRS):
        idx[k], micro[k] = p.micro(int(nuc[k]), float(E[k]))
        macro[k] = p.macro(int(mat[k]), float(E[k]))
        binv[k] = p.hash_bin(float(E[k]))
    return p, dict(
        kind=kind, bins=bins, pairs=PAIRS, input_seed=1000 + kind,
        library_checksum=f"{p.library_checksum():016x}", hash_checksum=f"{p.hash_checksum():016x}",
        bin_sha256=digest(binv), index_sha256=digest(idx), micro_sha256=digest(micro),
        macro_sha256=digest(macro),
        first=[dict(nuc=int(nuc[k]), mat=int(mat[k]), E=hexbits(E[k]), bin=int(binv[k]), idx=int(idx[k]),
                    micro=[hexbits(v) for v in micro[k]], macro=[hexbits(v) for v in macro[k]])
               for k in range(16)],
    )


def rng_vectors():
    L = O.lib()
    out = {"particle_streams": {}, "future_seed": []}
    for pid in (1, 2, 1_000_000, 1_000_000_000):
        s = O.C.c_uint64(L.orc_particle_seed(1, pid)) if hasattr(O, "C") else None
        import ctypes
        s = ctypes.c_uint64(L.orc_particle_seed(1, pid))
        out["particle_streams"][str(pid)] = [hexbits(L.orc_prn(ctypes.byref(s))) for _ in range(16)]
    for n, seed in ((0, 7), (1, 7), (152917, 1), (10**12, 99), (2**63 + 5, 3)):
        out["future_seed"].append([str(n), str(seed), str(L.orc_future_seed(n, seed))])
    xs = [1e-300, 1e-10, 0.0253, 0.5, 1.0, 1.5, 2.0, 10.0, 1e5, 2e7, 1e300]
    out["log"] = [[hexbits(x), hexbits(L.orc_log(x))] for x in xs]
    ys = [-700.0, -20.0, -1.0, -1e-9, 0.0, 1e-9, 0.5, 1.0, 28.3, 700.0]
    out["exp"] = [[hexbits(y), hexbits(L.orc_exp(y))] for y in ys]
    return out


def transport_vectors():
    """C1 (pin cell): 10000 histories x 4 batches (2 inactive), seed 1."""
    p = O.Problem(O.PINCELL, 1234, 4000)
    res, tally, recs = p.run(10_000, 4, 2, seed=1, threads=0, record_batch=1, record_n=1000)
    r = O.records_array(recs, 1000)
    return dict(
        problem="pincell", n_particles=10_000, n_batches=4, n_inactive=2, seed=1,
        k_coll=[hexbits(res.k_coll[b]) for b in range(4)],
        k_abs=[hexbits(res.k_abs[b]) for b in range(4)],
        k_track=[hexbits(res.k_track[b]) for b in range(4)],
        n_sites=[int(res.n_sites[b]) for b in range(4)],
        n_events=[int(x) for x in res.n_events], n_leaked=int(res.n_leaked), n_absorbed=int(res.n_absorbed),
        tally_sha256=digest(tally),
        records_batch=1, records_n=1000,
        records_counts_sha256=digest(np.stack([r[f] for f in ("n_xs", "n_adv", "n_cross", "n_coll", "n_sites",
                                                              "term")])),
        records_state_sha256=digest(r["e_final"], r["x_final"]),
        first_records=[[int(r[f][k]) for f in ("n_xs", "n_adv", "n_cross", "n_coll", "n_sites", "term")]
                       for k in range(10)],
    )


def main():
    O.build()
    ref = os.path.join(ROOT, "oracle", "_ref", "ref_rng")
    if os.path.exists(ref):
        out = json.loads(subprocess.run([ref], capture_output=True, text=True, check=True).stdout)
        out["source"] = "oracle/_ref/ref_rng built by oracle/build_ref.sh from /root/reference/proj/src/rng.hpp"
        with open(os.path.join(HERE, "ref_derive_seed.json"), "w") as f:
            json.dump(out, f, indent=1)
    with open(os.path.join(HERE, "oracle_rng.json"), "w") as f:
        json.dump(rng_vectors(), f, indent=1)
    lk = []
    for kind, bins in ((O.PINCELL, 4000), (O.ASSEMBLY, 4000), (O.ASSEMBLY, 100)):
        lk.append(lookup_vectors(kind, bins)[1])
    with open(os.path.join(HERE, "oracle_lookup.json"), "w") as f:
        json.dump(lk, f, indent=1)
    with open(os.path.join(HERE, "oracle_transport_c1.json"), "w") as f:
        json.dump(transport_vectors(), f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
