"""CPU emulation of the sm_100a pass kernel's dataflow, driven by the very
host tables the C planner builds (tcfftPlanTables / tcfftDescribePlan).

Test infrastructure: it lets the CPU suite check every index map (stage-1
gather addresses, writer destinations in the MN-major A operand, twiddle
tables, DFT block matrices, 128B-swizzled staging, output addresses) end to
end without a GPU, and measures shared-memory bank conflicts of each access
pattern.  The tcgen05 operand layouts it assumes (K-major B, MN-major A with
padded SBO, A-from-TMEM packing) are the ones tests/native/umma_probe.cu
verifies on the hardware.
"""

from __future__ import annotations

import numpy as np

from paper_2104_11471_b200 import _lib

ROW_DT = np.dtype([("gbase", "<i4"), ("addr", "<i4"), ("mp", "<i4"), ("tw", "<i4"), ("cr", "<f4"),
                   ("ci", "<f4"), ("wr", "<f4"), ("wi", "<f4")])


class PassTables:
    def __init__(self, dims, nx, ny, batch, index, dist=None, fused=False):
        # dist = (rank, world): a pass of the distributed single-transform plan
        if dist is None:
            desc = _lib.describe(dims, nx, ny, batch)
            rows, b, t = _lib.plan_tables(dims, nx, ny, batch, index)
        else:
            desc = _lib.describe_dist(nx, *dist, fused=fused)
            rows, b, t = _lib.dist_plan_tables(nx, *dist, index, fused=fused)
        self.d = desc["passes"][index]
        S, tm = len(self.d["stages"]), self.d["tiles_max"]
        self.rows = np.frombuffer(rows, dtype=ROW_DT).reshape(S, tm, 128)
        self.b = np.frombuffer(b, dtype=np.float16)
        self.t = np.frombuffer(t, dtype=np.float32) if len(t) else np.zeros(0, np.float32)

    def bmat(self, s):
        st = self.d["stages"][s]
        KP, NP = st["KP"], st["NP"]
        R = st["R"]
        k = np.arange(KP)[:, None]
        n = np.arange(NP)[None, :]
        off = (k // 16) * 32 * NP + (n % 8) * 16 + (n // 8) * 256 + ((k % 16) // 8) * 128 + (k % 8) * 2
        return self.b[(st["b_off"] + off) // 2].astype(np.float64)  # (KP, NP)


def _swz(b, mask):
    return b ^ ((b >> 3) & mask)


def _half(x):
    with np.errstate(over="ignore"):
        return np.asarray(x, dtype=np.float32).astype(np.float16)


def emulate_chunk(pt: PassTables, chunk_words: np.ndarray, stats: dict | None = None,
                  tw4_base: int = 0) -> np.ndarray:
    """chunk_words: (L,) uint32 interleaved fp16 pairs in linear staging order.
    Returns the (L,) uint32 output staging in linear order.  tw4_base: first
    global column of the strip (four-step pass 1 twiddle)."""
    d = pt.d
    swz, swz_out = d["swz_in"], d["swz_out"]
    L = len(chunk_words)
    stages = d["stages"]
    S = len(stages)
    lin = np.arange(L, dtype=np.int64) * 4
    sbuf = np.zeros(L, np.uint32)
    sbuf[_swz(lin, swz) // 4] = chunk_words

    # ---- stage 1 gather -> A (TMEM), interleaved K
    st = stages[0]
    R, T1, KP = st["R"], st["tiles"], st["KP"]
    rec = pt.rows[0, :T1]
    addr = (rec["gbase"][..., None].astype(np.int64) + np.arange(R) * d["gstride"]) * 4
    phys = _swz(addr, swz)
    if stats is not None:
        _bank_stats(stats, "gather_lds32", phys, 4)
    w = sbuf[phys // 4]  # (T1, 128, R)
    pairs = w.view(np.float16).reshape(T1, 128, R, 2).astype(np.float64)
    A = np.zeros((T1, 128, KP))
    if d.get("planar0"):  # radix-64 first stage: K = (re_0..re_R-1, im_0..im_R-1)
        A[..., :R] = pairs[..., 0]
        A[..., R: 2 * R] = pairs[..., 1]
    else:  # K = (re_0, im_0, re_1, im_1, ..)
        A[..., : 2 * R] = pairs.reshape(T1, 128, 2 * R)
    D = A @ pt.bmat(0)

    abuf = None
    for s in range(S - 1):
        st, nx_ = stages[s], stages[s + 1]
        R, Rn, T = st["R"], nx_["R"], st["tiles"]
        rec = pt.rows[s, :T]
        xr = D[..., :R].astype(np.float32)
        xi = D[..., R: 2 * R].astype(np.float32)
        # kernel: output j gets c * w^j (register recurrence; c = 1 at stage 1)
        c = (rec["cr"] + 1j * rec["ci"]) if s > 0 else np.ones(rec.shape)
        w = rec["wr"] + 1j * rec["wi"]
        tw = (c[..., None] * w[..., None] ** np.arange(R)).astype(np.complex64)
        trr, tii = tw.real, tw.imag
        yr = xr * trr - xi * tii
        yi = xr * tii + xi * trr
        hr, hi = _half(yr), _half(yi)
        abytes = nx_["tiles"] * nx_["tile_bytes"]
        abuf = np.zeros(abytes // 2, np.float16)
        a0 = rec["addr"].astype(np.int64)
        st_addr = []
        for h in range(R // 8):
            base = a0 + h * st["hstep"]
            st_addr.append(base)
            st_addr.append(base + st["im_off"])
            for j8 in range(8):
                j = 8 * h + j8
                abuf[(base + j8 * 2) // 2] = hr[..., j]
                abuf[(base + st["im_off"] + j8 * 2) // 2] = hi[..., j]
        if stats is not None:
            _bank_stats(stats, "writer_sts128", np.stack(st_addr, -1), 16)
        # next stage: A (MN-major, split planes), D = A @ B
        Tn, KPn, sbo, tb = nx_["tiles"], nx_["KP"], nx_["sbo"], nx_["tile_bytes"]
        t = np.arange(Tn)[:, None, None]
        row = np.arange(128)[None, :, None]
        k = np.arange(KPn)[None, None, :]
        off = t * tb + (row // 8) * sbo + (row % 8) * 2 + k * 16
        A = abuf[off // 2].astype(np.float64)
        D = A @ pt.bmat(s + 1)

    st = stages[S - 1]
    R, T = st["R"], st["tiles"]
    rec = pt.rows[S - 1, :T]
    yr, yi = D[..., :R].astype(np.float32), D[..., R: 2 * R].astype(np.float32)
    if d["tw4_total"]:
        # kernel: c4 = A[k] * W^{tr k} (host), w4 = r * W^{tr s} (host); A, r per chunk
        Nt, s_ = d["tw4_total"], d["N"] // R
        A = np.exp(-2j * np.pi * ((tw4_base * rec["mp"].astype(np.int64)) % Nt) / Nt)
        r = np.exp(-2j * np.pi * ((tw4_base * s_) % Nt) / Nt)
        c4 = A * (rec["cr"] + 1j * rec["ci"])
        w4 = r * (rec["wr"] + 1j * rec["wi"])
        tw = (c4[..., None] * w4[..., None] ** np.arange(R)).astype(np.complex64)
        yr, yi = yr * tw.real - yi * tw.imag, yr * tw.imag + yi * tw.real
    hr, hi = _half(yr), _half(yi)
    words = np.stack([hr, hi], -1).view(np.uint32)[..., 0]  # (T,128,R)
    oaddr = (rec["addr"][..., None].astype(np.int64) + np.arange(R) * d["ostride"]) * 4
    ophys = _swz(oaddr, swz_out)
    if stats is not None:
        _bank_stats(stats, "final_sts32", ophys, 4)
    if d["kind"] == "stripT" and d["pitch"] != d["N"]:  # rows at a padded pitch, written back row by row
        Lo = d["T"] * d["pitch"]
        obuf = np.zeros(Lo, np.uint32)
        obuf[ophys // 4] = words
        assert len(np.unique(ophys)) == ophys.size, "output staging addresses collide"
        return obuf.reshape(d["T"], d["pitch"])[:, : d["N"]].reshape(-1)
    obuf = np.zeros(L, np.uint32)
    obuf[ophys // 4] = words
    assert len(np.unique(ophys)) == ophys.size, "output staging addresses collide"
    return obuf[_swz(lin, swz_out) // 4]


def _bank_stats(stats, name, addrs, width):
    """addrs: (..., 128 lanes, n_instr) byte addresses of one access each.
    Counts shared-memory wavefronts per warp instruction."""
    a = np.asarray(addrs)
    a = a.reshape(-1, 128, a.shape[-1]) if a.ndim >= 3 else a.reshape(1, 128, -1)
    lanes_per_phase = 32 if width <= 4 else (16 if width == 8 else 8)
    tot = cnt = 0
    for tile in a:
        for w in range(4):
            warp = tile[32 * w: 32 * w + 32]
            for ins in range(warp.shape[1]):
                wf = 0
                for p0 in range(0, 32, lanes_per_phase):
                    words = set()
                    for lane in range(p0, p0 + lanes_per_phase):
                        for b in range(0, width, 4):
                            words.add(int(warp[lane, ins]) + b)
                    banks = {}
                    for x in words:
                        banks.setdefault((x // 4) % 32, set()).add(x // 4)
                    wf += max(len(v) for v in banks.values())
                tot += wf
                cnt += 1
    ideal = 1 if width <= 4 else (2 if width == 8 else 4)
    s = stats.setdefault(name, [0, 0, ideal])
    s[0] += tot
    s[1] += cnt


def run_pass_row(pt: PassTables, pairs: np.ndarray, stats=None) -> np.ndarray:
    """pairs: (count, N, 2) fp16 contiguous transforms."""
    N, T, E, P = pt.d["N"], pt.d["T"], pt.d["E"], pt.d["pitch"]
    count = pairs.shape[0]
    words = np.ascontiguousarray(pairs).view(np.uint32).reshape(count, N)
    out = np.empty_like(words)
    for c in range(0, count, T):
        nt = min(T, count - c)
        w = np.zeros((T, P), np.uint32)
        w[:nt, :N] = words[c: c + nt]
        o = emulate_chunk(pt, w.reshape(-1), stats if c == 0 else None).reshape(T, P)
        out[c: c + nt] = o[:nt, :N]
    return out.view(np.float16).reshape(pairs.shape)


def run_pass_strip(pt: PassTables, img: np.ndarray, stats=None) -> np.ndarray:
    """img: (images, nx, ny, 2) fp16; column FFTs of length nx."""
    d = pt.d
    C, IMG = d["C"], d["IMG"]
    B, nx, ny, _ = img.shape
    words = np.ascontiguousarray(img).view(np.uint32)[..., 0]  # (B, nx, ny)
    out = np.empty_like(words)
    first = True
    for b0 in range(0, B, IMG):
        for c0 in range(0, ny, C):
            blk = np.zeros((IMG, nx, C), np.uint32)
            nb = min(IMG, B - b0)
            blk[:nb] = words[b0: b0 + nb, :, c0: c0 + C]
            o = emulate_chunk(pt, blk.reshape(-1), stats if first else None, tw4_base=c0).reshape(IMG, nx, C)
            first = False
            out[b0: b0 + nb, :, c0: c0 + C] = o[:nb]
    return out[..., None].view(np.float16).reshape(img.shape)


def run_pass_rowT(pt: PassTables, rows: np.ndarray, images: int) -> np.ndarray:
    """Four-step pass 2: rows (images*N1, N2, 2) fp16 -> out (images, N2, N1, 2)
    (row k1 of image b lands in column k1 of the transposed output)."""
    N, T, P = pt.d["N"], pt.d["T"], pt.d["pitch"]
    count = rows.shape[0]
    n1 = count // images
    words = np.ascontiguousarray(rows).view(np.uint32).reshape(count, N)
    out = np.zeros((images, N, n1), np.uint32)
    for c in range(0, count, T):
        w = np.zeros((T, P), np.uint32)
        w[:, :N] = words[c: c + T]
        o = emulate_chunk(pt, w.reshape(-1))[: T * N].reshape(N, T)
        b, k0 = c // n1, c % n1
        out[b, :, k0: k0 + T] = o
    return out[..., None].view(np.float16).reshape(images, N, n1, 2)


def run_fourstep(n: int, pairs: np.ndarray) -> np.ndarray:
    """Full four-step 1D transform (both passes) of (B, n, 2) fp16."""
    B = pairs.shape[0]
    p1 = PassTables(1, n, 0, B, 0)
    p2 = PassTables(1, n, 0, B, 1)
    n1, n2 = p1.d["N"], p2.d["N"]
    y = run_pass_strip(p1, pairs.reshape(B, n1, n2, 2))
    z = run_pass_rowT(p2, y.reshape(B * n1, n2, 2), B)
    return z.reshape(B, n, 2)


def run_threestep(n: int, pairs: np.ndarray) -> np.ndarray:
    """Three-pass 1D transform (N >= 2^19) of (B, n, 2) fp16, pass by pass as
    the planner lays it out (plan.cpp build_three_step)."""
    B = pairs.shape[0]
    pa, pb, pc = (PassTables(1, n, 0, B, i) for i in range(3))
    N1, N2, N3 = pa.d["N"], pb.d["N"], pc.d["N"]
    shift = pb.d["tw4_shift"]
    x = np.ascontiguousarray(pairs).view(np.uint32).reshape(B, N1, N2 * N3)
    # pass A: column strips of [N1][N2 N3], each column -> a contiguous row [col][k1]
    C = pa.d["C"]
    y1 = np.empty((B, N2 * N3, N1), np.uint32)
    for b in range(B):
        for c0 in range(0, N2 * N3, C):
            o = emulate_chunk(pa, np.ascontiguousarray(x[b, :, c0: c0 + C]).reshape(-1), tw4_base=c0)
            y1[b, c0: c0 + C] = o.reshape(C, N1)
    # pass B: column strips of [N2][N3 N1] in place, twiddle exponent (col >> shift) k2
    y = y1.reshape(B, N2, N3 * N1)
    C = pb.d["C"]
    y2 = np.empty_like(y)
    for b in range(B):
        for c0 in range(0, N3 * N1, C):
            o = emulate_chunk(pb, np.ascontiguousarray(y[b, :, c0: c0 + C]).reshape(-1), tw4_base=c0 >> shift)
            y2[b, :, c0: c0 + C] = o.reshape(N2, C)
    # pass C: strips of each [N3][N1] image k2 -> X[b][k3][k2][k1]
    y = y2.reshape(B, N2, N3, N1)
    C = pc.d["C"]
    out = np.empty((B, N3, N2, N1), np.uint32)
    for b in range(B):
        for k2 in range(N2):
            for c0 in range(0, N1, C):
                o = emulate_chunk(pc, np.ascontiguousarray(y[b, k2, :, c0: c0 + C]).reshape(-1))
                out[b, :, k2, c0: c0 + C] = o.reshape(N3, C)
    return out.reshape(B, n)[..., None].view(np.float16).reshape(B, n, 2)


def run_twopass_blocked(n: int, pairs: np.ndarray) -> np.ndarray:
    """Two-pass 1D transform (2^19 <= N <= 2^22, plan.cpp build_two_pass_blocked)
    of (B, n, 2) fp16: pass 1 column strips of [N1][N2] + twiddle, each chunk's
    [k1][C] staging tile stored contiguously (workspace Y[b][n2 / C][k1][n2 % C]);
    pass 2 rows k1 of the blocked workspace (T rows of every block per chunk),
    transposed store X[k1 + N1 k2]."""
    B = pairs.shape[0]
    p1, p2 = PassTables(1, n, 0, B, 0), PassTables(1, n, 0, B, 1)
    assert p2.d["kind"] == "rowTB", p2.d["kind"]
    N1, N2, C, T = p1.d["N"], p2.d["N"], p1.d["C"], p2.d["T"]
    x = np.ascontiguousarray(pairs).view(np.uint32).reshape(B, N1, N2)
    y = np.empty((B, N2 // C, N1, C), np.uint32)
    for b in range(B):
        for cb in range(N2 // C):
            o = emulate_chunk(p1, np.ascontiguousarray(x[b, :, cb * C: (cb + 1) * C]).reshape(-1), tw4_base=cb * C)
            y[b, cb] = o.reshape(N1, C)
    out = np.empty((B, N2, N1), np.uint32)
    for b in range(B):
        for r0 in range(0, N1, T):
            w = np.ascontiguousarray(y[b, :, r0: r0 + T, :]).reshape(-1)  # staging [block][T][C]
            out[b, :, r0: r0 + T] = emulate_chunk(p2, w).reshape(N2, T)
    return out.reshape(B, n)[..., None].view(np.float16).reshape(B, n, 2)


def run_2d_split(nx: int, ny: int, pairs: np.ndarray) -> np.ndarray:
    """2D transform with split columns (nx >= 8192, plan.cpp
    build_2d_split_columns) of (B, nx*ny, 2) fp16: the row pass, then pass 2a
    (length-N1 column strips of [N1][N2 ny] + twiddle, exponent (c >> log2 ny) k1)
    and pass 2b (strips of each [N2][ny] image (b, k1), stored to row k1 + N1 k2)."""
    B = pairs.shape[0]
    p0, pa, pb = (PassTables(2, nx, ny, B, i) for i in range(3))
    assert p0.d["kind"] == "row" and pa.d["kind"] == "strip" and pb.d["kind"] == "strip"
    rows = run_pass_row(p0, pairs.reshape(B * nx, ny, 2))
    N1, N2, shift = pa.d["N"], pb.d["N"], pa.d["tw4_shift"]
    x = np.ascontiguousarray(rows).view(np.uint32).reshape(B, N1, N2 * ny)
    C = pa.d["C"]
    y = np.empty_like(x)
    for b in range(B):
        for c0 in range(0, N2 * ny, C):
            o = emulate_chunk(pa, np.ascontiguousarray(x[b, :, c0: c0 + C]).reshape(-1), tw4_base=c0 >> shift)
            y[b, :, c0: c0 + C] = o.reshape(N1, C)
    y = y.reshape(B, N1, N2, ny)
    C = pb.d["C"]
    out = np.empty((B, N2, N1, ny), np.uint32)  # row k1 + N1 k2 = [k2][k1]
    for b in range(B):
        for k1 in range(N1):
            for c0 in range(0, ny, C):
                o = emulate_chunk(pb, np.ascontiguousarray(y[b, k1, :, c0: c0 + C]).reshape(-1))
                out[b, :, k1, c0: c0 + C] = o.reshape(N2, C)
    return out.reshape(B, nx * ny)[..., None].view(np.float16).reshape(B, nx * ny, 2)


class EmulatedDistLocal:
    """The local steps of paper_2104_11471_b200.dist.DistPlan replayed on the
    CPU from the planner's own tables (tcfftDistPlanTables): lets CPU ranks
    (gloo) run the distributed transform end to end."""

    def __init__(self, nx, rank, world):
        self.p0 = PassTables(1, nx, 0, 1, 0, dist=(rank, world))
        self.p1 = PassTables(1, nx, 0, 1, 1, dist=(rank, world))
        self.world = world

    def pass0(self, slab):
        import torch

        d = self.p0.d
        n1, C, col0 = d["N"], d["C"], d["tw4_col0"]
        w = slab.numpy().view(np.uint32).reshape(n1, -1)
        out = np.empty_like(w)
        for c0 in range(0, w.shape[1], C):
            o = emulate_chunk(self.p0, np.ascontiguousarray(w[:, c0: c0 + C]).reshape(-1), tw4_base=col0 + c0)
            out[:, c0: c0 + C] = o.reshape(n1, C)
        return torch.from_numpy(out.view(np.float16).reshape(slab.shape))

    def unpack(self, recv, rows):
        n2 = self.p1.d["N"]
        G = self.world
        r = recv.reshape(G, -1, n2 // G, 2)  # [G][N1/G][N2/G]
        rows.copy_(r.permute(1, 0, 2, 3).reshape(rows.shape))
        return rows

    def pass1(self, rows, out):
        import torch

        n2 = self.p1.d["N"]
        x = rows.numpy().reshape(-1, n2, 2)
        y = run_pass_rowT(self.p1, x, 1)  # (1, N2, N1/G, 2)
        out.copy_(torch.from_numpy(np.ascontiguousarray(y)).reshape(out.shape))
        return out


class EmulatedDistLocalFused:
    """The fused distributed plan's local steps replayed on the CPU
    (tcfftDistPlanTablesFused): pass 0 returns the N1/G-row slices of every
    staging tile, arranged [G][blocks][N1/G][C] (what the kernel's peer stores
    deliver to each rank); pass 1 is the blocked-rows pass over the received
    [N2/C][N1/G][C] buffer."""

    fused = True

    def __init__(self, nx, rank, world):
        self.p0 = PassTables(1, nx, 0, 1, 0, dist=(rank, world), fused=True)
        self.p1 = PassTables(1, nx, 0, 1, 1, dist=(rank, world), fused=True)
        self.world = world
        assert self.p1.d["kind"] == "rowTB"

    def pass0(self, slab):
        import torch

        d = self.p0.d
        n1, C, col0 = d["N"], d["C"], d["tw4_col0"]
        G = self.world
        w = slab.numpy().view(np.uint32).reshape(n1, -1)
        nb = w.shape[1] // C
        send = np.empty((G, nb, n1 // G, C), np.uint32)
        for cb in range(nb):
            o = emulate_chunk(self.p0, np.ascontiguousarray(w[:, cb * C: (cb + 1) * C]).reshape(-1),
                              tw4_base=col0 + cb * C).reshape(n1, C)
            send[:, cb] = o.reshape(G, n1 // G, C)
        return torch.from_numpy(send.reshape(-1)[..., None].view(np.float16).reshape(-1, 2))

    def pass1(self, recv, out):
        import torch

        C, T, n2 = self.p0.d["C"], self.p1.d["T"], self.p1.d["N"]
        y = recv.numpy().view(np.uint32).reshape(n2 // C, -1, C)  # [blocks][N1/G][C]
        rows = y.shape[1]
        res = np.empty((n2, rows), np.uint32)
        for r0 in range(0, rows, T):
            wv = np.ascontiguousarray(y[:, r0: r0 + T, :]).reshape(-1)
            res[:, r0: r0 + T] = emulate_chunk(self.p1, wv).reshape(n2, T)
        out.copy_(torch.from_numpy(res.reshape(-1)[..., None].view(np.float16).reshape(out.shape)))
        return out
