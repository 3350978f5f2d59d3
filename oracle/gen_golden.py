"""Generate tests/golden/*.npz by running the REFERENCE implementation itself.

TEST INFRASTRUCTURE ONLY (see oracle/restate.py header).  Run in the build
container, where the read-only reference lives:

    python oracle/gen_golden.py [--ref /root/reference/pkg/src] [--ext baseline/_ref]

The reference is imported as-is (``tcfft`` package, reference
``pkg/src/tcfft/__init__.py``).  Small cases run its pure-python MMA backend
(``TCFFT_BACKEND=py``, ``backend.py:33-45``); the large hash-only cases (1D
2^17 .. 2^24, 2D 1024x512 .. 4096^2) run its compiled Cython backend
(``TCFFT_BACKEND=ext``, ``_core.pyx``) from the unmodified install in
``baseline/_ref`` (``pip install --no-deps --target baseline/_ref`` of a copy
of ``/root/reference/pkg``), which the reference's own tests prove
bit-identical to the python one (``tests/test_backends.py:30-60``).  Cases run
in parallel worker processes (one reference process per case).
Inputs follow the reference CLI protocol (seeded U[-1,1) re/im rounded to fp16,
``cli.py:40-43``).  Outputs are stored as raw fp16 pairs; large cases store a
SHA-256 of the output bytes instead of the bytes.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
sys.path.insert(0, str(ROOT))

from oracle.restate import random_pairs  # noqa: E402

# (kind, nx, ny, batch, seed-config-id)
CASES_1D = [(n, b) for n, b in [
    (2, 3), (4, 3), (8, 3), (16, 3), (32, 3), (64, 3), (128, 3), (256, 4),
    (512, 3), (1024, 2), (2048, 2), (4096, 2), (8192, 1), (16384, 1),
    (32768, 1), (65536, 1)]]
CASES_2D = [(2, 2, 2), (16, 16, 2), (32, 64, 1), (64, 32, 1), (256, 256, 1),
            (512, 256, 1)]
# large cases: SHA-256 only (the reference's ext backend; minutes each)
CASES_1D_BIG = [(1 << k, 1) for k in range(17, 25)]
CASES_2D_BIG = [(1024, 512, 1), (1024, 1024, 1), (2048, 2048, 1), (4096, 4096, 1)]
STORE_LIMIT = 1 << 15  # elements per case stored verbatim; above: hash only


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint16).tobytes()).hexdigest()


def _run_case(job):
    """One reference execution in a fresh worker process (job = (tag, nx, ny,
    batch, cfg, backend, src))."""
    tag, nx, ny, batch, cfg, backend, src = job
    os.environ["TCFFT_BACKEND"] = backend
    sys.path.insert(0, src)
    import tcfft  # the reference package

    assert tcfft.backend.active_backend() == backend, (tcfft.__file__, backend)
    total = nx * (ny or 1)
    x = random_pairs([cfg, 0], batch, total)
    data = tcfft.BatchedTensor(x.reshape(-1, 2).copy(), batch, total)
    plan = tcfft.plan_1d(nx, batch) if ny is None else tcfft.plan_2d(nx, ny, batch)
    tcfft.execute(plan, data)
    y = data.pairs.reshape(batch, total, 2)
    return f"{tag}|{nx}|{ny or 0}|{batch}|{cfg}|{_sha(y)}", (y if batch * total <= STORE_LIMIT else None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--ext", default=str(ROOT / "baseline" / "_ref"))
    ap.add_argument("--out", default=str(ROOT / "tests" / "golden"))
    ap.add_argument("--jobs", type=int, default=len(os.sched_getaffinity(0)))
    args = ap.parse_args()
    import multiprocessing as mp

    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    store = {}
    meta = []
    jobs = [("1d", n, None, b, 100 + i, "py", args.ref) for i, (n, b) in enumerate(CASES_1D)]
    jobs += [("2d", nx, ny, b, 200 + i, "py", args.ref) for i, (nx, ny, b) in enumerate(CASES_2D)]
    jobs += [("1d", n, None, b, 300 + i, "ext", args.ext) for i, (n, b) in enumerate(CASES_1D_BIG)]
    jobs += [("2d", nx, ny, b, 400 + i, "ext", args.ext) for i, (nx, ny, b) in enumerate(CASES_2D_BIG)]
    # longest first, so the pool's tail is short
    order = sorted(range(len(jobs)), key=lambda i: -jobs[i][1] * (jobs[i][2] or 1) * jobs[i][3])
    with mp.get_context("spawn").Pool(args.jobs, maxtasksperchild=1) as pool:
        res = dict(zip(order, pool.map(_run_case, [jobs[i] for i in order], chunksize=1)))
    for i, job in enumerate(jobs):
        rec, y = res[i]
        meta.append(rec)
        if y is not None:
            store[f"{job[0]}_{job[1]}_{job[2] or 0}_out"] = y
        print(rec, flush=True)

    os.environ["TCFFT_BACKEND"] = "py"
    sys.path.insert(0, args.ref)
    import tcfft  # the reference package (KATs below)

    # Known-answer vectors from the reference's own tests.
    kat = {}
    z = np.zeros((1, 16, 2), np.float16)
    z[0, 0, 0] = 1
    d = tcfft.BatchedTensor(z.reshape(-1, 2).copy(), 1, 16)
    tcfft.execute(tcfft.plan_1d(16, 1), d)  # test_executor.py:87-92
    kat["impulse16_out"] = d.pairs.reshape(1, 16, 2)
    n = 256
    tone = np.exp(-2j * np.pi * 5 * np.arange(n) / n)
    tz = np.empty((1, n, 2), np.float16)
    tz[0, :, 0] = tone.real.astype(np.float16)
    tz[0, :, 1] = tone.imag.astype(np.float16)
    d = tcfft.BatchedTensor(tz.reshape(-1, 2).copy(), 1, n)
    tcfft.execute(tcfft.plan_1d(n, 1), d)  # test_executor.py:95-103
    kat["tone256_in"] = tz
    kat["tone256_out"] = d.pairs.reshape(1, n, 2)
    z2 = np.zeros((1, 256, 2), np.float16)
    z2[0, 0, 0] = 1
    d = tcfft.BatchedTensor(z2.reshape(-1, 2).copy(), 1, 256)
    tcfft.execute(tcfft.plan_2d(16, 16, 1), d)  # test_executor.py:160-165
    kat["impulse2d16_out"] = d.pairs.reshape(1, 256, 2)

    np.savez_compressed(out / "reference_outputs.npz", meta=np.array(meta), **store, **kat)
    print("wrote", out / "reference_outputs.npz")


if __name__ == "__main__":
    main()
