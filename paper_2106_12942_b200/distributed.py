"""Multi-GPU RHSEG: the quadrant recursion sharded by subtrees.

Sections at every level are independent until their parent's stitch
(recursive.py:145-170), so with G ranks:

* l* = ceil(log4 G); the 4^l* sections of level top = l*+1 are subtree roots,
  dealt out in contiguous row-major ranges (each rank's range is a rectangle of
  the level-top grid);
* every rank runs levels L..top of its subtrees locally (one batched
  rhseg_run_subtrees call; no communication);
* ONE exchange: the level-top section states (counts, band sums, adjacency,
  pixel assignment -- what stitch needs, sections.py:103-163) are gathered to
  rank 0 over NCCL, which runs levels top-1..1 (negligible at t=16);
* merge logs stay on the ranks' devices until the result is assembled; they are
  gathered the same way and put into the reference's canonical log order
  (level L..1, row-major over the whole grid; recursive.py:95-104).

Results are GPU-count invariant by construction (each section's merges depend
only on its own inputs). Host logic (plan, log reassembly) is pure Python so it
is covered by gloo world-size-2 tests on CPU.
"""

from __future__ import annotations

import ctypes
import json
import time

import numpy as np

from . import _lib


# ---------------------------------------------------------------------------
# plan (pure host logic)
# ---------------------------------------------------------------------------
def shard_plan(levels: int, world: int):
    """-> (top_level, [(r0, c0, nr, nc) per rank] or None for an idle rank).

    top_level = l*+1 with l* the smallest l such that 4^l >= world, capped at
    `levels`; subtree k (row-major over the 2^l* x 2^l* grid) goes to rank
    floor(k * world / S) so ranges are contiguous; every range must be a
    rectangle (true for world in {1, 2, 4, 8, 16, ...})."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if world == 1 or levels == 1:
        return 1, [(0, 0, 1, 1)] + [None] * (world - 1)
    lstar = 0
    while 4 ** lstar < world:
        lstar += 1
    top = min(lstar + 1, levels)
    side = 1 << (top - 1)
    S = side * side
    blocks = []
    for g in range(world):
        a, b = g * S // world, (g + 1) * S // world
        if a == b:
            blocks.append(None)
            continue
        if a // side == (b - 1) // side:
            blocks.append((a // side, a % side, 1, b - a))
        elif a % side == 0 and b % side == 0:
            blocks.append((a // side, 0, (b - a) // side, side))
        else:
            raise ValueError(f"world={world}: subtree range [{a},{b}) is not a rectangle of the {side}x{side} grid")
    return top, blocks


def block_sections(block, level: int, top: int):
    """Section ids (level, row, col) of `block` at `level` >= top, row-major."""
    r0, c0, nr, nc = block
    s = 1 << (level - top)
    return [(level, r0 * s + r, c0 * s + c) for r in range(nr * s) for c in range(nc * s)]


def assemble_logs(levels: int, parts):
    """Canonical log order from per-rank pieces.

    parts: iterable of (sections, survivor, absorbed, dissim, kind) where
    sections is a list of (level, row, col, offset, count) into that part's
    flat arrays. Returns (section_ids, a, b, d, k) concatenated level L..1,
    row-major (recursive.py:95-104 log_order)."""
    where = {}
    for pi, (secs, *_rest) in enumerate(parts):
        for lev, row, col, off, cnt in secs:
            key = (int(lev), int(row), int(col))
            if key in where:
                raise ValueError(f"section {key} reported twice")
            where[key] = (pi, int(off), int(cnt))
    parts = list(parts)
    order = sorted(where, key=lambda k: (-k[0], k[1], k[2]))
    ids, pa, pb, pd, pk = [], [], [], [], []
    for key in order:
        pi, off, cnt = where[key]
        _, a, b, d, k = parts[pi]
        ids.append((key, cnt))
        pa.append(np.asarray(a[off:off + cnt]))
        pb.append(np.asarray(b[off:off + cnt]))
        pd.append(np.asarray(d[off:off + cnt]))
        pk.append(np.asarray(k[off:off + cnt]))
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt))
    return ids, cat(pa, np.int32), cat(pb, np.int32), cat(pd, np.float64), cat(pk, np.uint8)


# ---------------------------------------------------------------------------
# device side (one rank)
# ---------------------------------------------------------------------------
class RankRunner:
    """One rank's part of a sharded RHSEG on its own device/context."""

    def __init__(self, params_c, edge: int, bands: int, levels: int, device: int, private_ctx: bool = False):
        self.p = params_c
        self.edge, self.bands, self.levels = edge, bands, levels
        self.ctx = _lib.Context(device) if private_ctx else _lib.context(device)
        self.lib = _lib.load()

    def run_block(self, cube_ptr: int, top: int, block, stream: int | None):
        r0, c0, nr, nc = block
        _lib.check(self.lib.rhseg_run_subtrees(self.ctx.handle, ctypes.c_void_p(cube_ptr), self.edge, self.bands,
                                               ctypes.byref(self.p), top, r0, c0, nr, nc,
                                               ctypes.c_void_p(stream) if stream else None), "rhseg_run_subtrees")

    def top_info(self):
        nsec, rp, se = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _lib.check(self.lib.rhseg_top_info(self.ctx.handle, ctypes.byref(nsec), ctypes.byref(rp), ctypes.byref(se),
                                           None, None), "rhseg_top_info")
        R0 = np.zeros(nsec.value, np.int32)
        nlog = np.zeros(nsec.value, np.int32)
        _lib.check(self.lib.rhseg_top_info(self.ctx.handle, None, None, None, _lib.ptr(R0), _lib.ptr(nlog)),
                   "rhseg_top_info")
        return nsec.value, rp.value, se.value, R0, nlog

    def pack_bytes(self, rp: int, sec_edge: int) -> int:
        n = ctypes.c_int64()
        _lib.check(self.lib.rhseg_pack_bytes(rp, self.bands, sec_edge, ctypes.byref(n)), "rhseg_pack_bytes")
        return n.value

    def export(self, rp: int, dptr: int, stream):
        _lib.check(self.lib.rhseg_export_top(self.ctx.handle, rp, ctypes.c_void_p(dptr),
                                             ctypes.c_void_p(stream) if stream else None), "rhseg_export_top")

    def run_upper(self, dptr: int, top: int, rp: int, R0, nlog, stream):
        R0 = np.ascontiguousarray(R0, np.int32)
        nlog = np.ascontiguousarray(nlog, np.int32)
        _lib.check(self.lib.rhseg_run_upper(self.ctx.handle, ctypes.c_void_p(dptr), top, rp, _lib.ptr(R0),
                                            _lib.ptr(nlog), self.edge, self.bands, ctypes.byref(self.p),
                                            ctypes.c_void_p(stream) if stream else None), "rhseg_run_upper")

    def sections(self):
        from .recursive import result_info

        info = result_info(self.ctx)
        ns = int(info.n_sections)
        lev, row, col = (np.zeros(ns, np.int32) for _ in range(3))
        off, cnt = np.zeros(ns, np.int64), np.zeros(ns, np.int64)
        _lib.check(self.lib.rhseg_result_sections(self.ctx.handle, _lib.ptr(lev), _lib.ptr(row), _lib.ptr(col),
                                                  _lib.ptr(off), _lib.ptr(cnt)), "rhseg_result_sections")
        return info, np.stack([lev, row, col, off, cnt], 1).astype(np.int64)

    def log_device(self, a_ptr, b_ptr, d_ptr, k_ptr, stream):
        vp = ctypes.c_void_p
        _lib.check(self.lib.rhseg_result_log_device(self.ctx.handle, vp(a_ptr), vp(b_ptr), vp(d_ptr), vp(k_ptr),
                                                    vp(stream) if stream else None), "rhseg_result_log_device")


def host_log_part(runner: RankRunner):
    """(sections, a, b, d, k) of a runner's last run, copied to the host."""
    info, secs = runner.sections()
    n = int(info.n_records)
    a, b = np.zeros(n, np.int32), np.zeros(n, np.int32)
    d, k = np.zeros(n, np.float64), np.zeros(n, np.uint8)
    _lib.check(runner.lib.rhseg_result_log(runner.ctx.handle, _lib.ptr(a), _lib.ptr(b), _lib.ptr(d), _lib.ptr(k)),
               "rhseg_result_log")
    return secs.tolist(), a, b, d, k


def emulate_sharded(image, params, world: int, device: int = 0, connectivity: int = 8):
    """The sharded data path of `world` ranks replayed on ONE device (one
    private context per rank, the gather replaced by a device concatenation).
    Used by the GPU tests to prove the partial-run / export / import /
    reassembly path bit-identical to the single-GPU run."""
    import torch

    from .recursive import B200Executor, RecordList, collect_result, result_info
    from .sections import SectionId

    edge, bands, levels = image.width, image.bands, params.levels
    pc = B200Executor(connectivity=connectivity, device=device).c_params(params)
    dev = torch.device("cuda", device)
    cube = torch.from_numpy(np.ascontiguousarray(image.samples, np.float32)).to(dev)
    top, blocks = shard_plan(levels, world)
    if top == 1:
        r = RankRunner(pc, edge, bands, levels, device, private_ctx=True)
        r.run_block(cube.data_ptr(), 1, (0, 0, 1, 1), None)
        return collect_result(r.ctx, result_info(r.ctx), edge, bands, levels)
    runners, metas, parts = [], [], []
    for blk in blocks:
        if blk is None:
            continue
        r = RankRunner(pc, edge, bands, levels, device, private_ctx=True)
        r.run_block(cube.data_ptr(), top, blk, None)
        runners.append(r)
        metas.append(r.top_info())
        parts.append(host_log_part(r))
    rpc = max(m[1] for m in metas)
    se = metas[0][2]
    pbytes = runners[0].pack_bytes(rpc, se)
    side = 1 << (top - 1)
    allp = torch.zeros(side * side * pbytes, dtype=torch.uint8, device=dev)
    k = 0
    for r, m in zip(runners, metas):
        n = m[0]
        tmp = torch.zeros(n * pbytes, dtype=torch.uint8, device=dev)
        r.export(rpc, tmp.data_ptr(), None)
        torch.cuda.synchronize(dev)
        allp[k * pbytes:(k + n) * pbytes].copy_(tmp)
        k += n
    torch.cuda.synchronize(dev)
    R0 = np.concatenate([m[3] for m in metas]).astype(np.int32)
    nlog = np.concatenate([m[4] for m in metas]).astype(np.int32)
    root = RankRunner(pc, edge, bands, levels, device, private_ctx=True)
    root.run_upper(allp.data_ptr(), top, rpc, R0, nlog, None)
    res = collect_result(root.ctx, result_info(root.ctx), edge, bands, levels)
    parts.append(host_log_part(root))
    ids, A, B, D, K = assemble_logs(levels, parts)
    logs, o = [], 0
    for (lev, row, col), cnt in ids:
        logs.append((SectionId(lev, row, col), RecordList(A[o:o + cnt], B[o:o + cnt], D[o:o + cnt], K[o:o + cnt])))
        o += cnt
    res.section_logs = logs
    return res


# ---------------------------------------------------------------------------
# NCCL step (torch.distributed plumbing; the data path is the C-ABI above)
# ---------------------------------------------------------------------------
class ShardedRhseg:
    """torch.distributed (NCCL) sharded RHSEG: call step(cube) on every rank."""

    def __init__(self, params, edge: int, bands: int, device: int, connectivity: int = 8):
        self.record = False  # keep this rank's lower-level phases/loop info (bench)
        self.last_block = None
        import torch
        import torch.distributed as dist

        from .recursive import B200Executor

        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.dev = torch.device("cuda", device)
        self.params = params
        self.levels = params.levels
        self.top, self.blocks = shard_plan(params.levels, self.world)
        self.block = self.blocks[self.rank]
        ex = B200Executor(connectivity=connectivity, device=device)
        self.runner = RankRunner(ex.c_params(params), edge, bands, params.levels, device)
        self.edge, self.bands = edge, bands
        self._bufs = {}
        # NCCL moves device buffers directly; gloo (CPU tests, several ranks on one
        # device) stages them through host memory
        self.host_comm = dist.get_backend() != "nccl"

    def _all_gather(self, out, t):
        if not self.host_comm:
            return self.dist.all_gather(out, t)
        tmp = [o.cpu() for o in out]
        self.dist.all_gather(tmp, t.cpu())
        for o, x in zip(out, tmp):
            o.copy_(x)

    def _gather(self, t, out):
        if not self.host_comm:
            return self.dist.gather(t, out, dst=0)
        tmp = [o.cpu() for o in out] if out is not None else None
        self.dist.gather(t.cpu(), tmp, dst=0)
        if out is not None:
            for o, x in zip(out, tmp):
                o.copy_(x)

    def _buf(self, name, n, dtype):
        t = self._bufs.get(name)
        if t is None or t.numel() < n:
            t = self.torch.empty(max(n, 1), dtype=dtype, device=self.dev)
            self._bufs[name] = t
        return t[:max(n, 1)]

    def step(self, cube, gather_logs: bool = True):
        """One sharded RHSEG over `cube` (device tensor, full image on every
        rank). Leaves the root result in rank 0's context; returns the gathered
        log pieces on rank 0 when gather_logs."""
        torch, dist = self.torch, self.dist
        stream = torch.cuda.current_stream(self.dev).cuda_stream
        if self.top == 1:
            if self.rank == 0:
                self.runner.run_block(cube.data_ptr(), 1, (0, 0, 1, 1), stream)
            return None
        side = 1 << (self.top - 1)
        S = side * side
        per = [0 if b is None else b[2] * b[3] for b in self.blocks]
        maxn = max(per)
        se = self.edge // side
        if self.block is not None:
            self.runner.run_block(cube.data_ptr(), self.top, self.block, stream)
            nsec, rp, _, R0, nlog = self.runner.top_info()
            if self.record:  # this rank's lower levels (the bench's per-rank roofline)
                self.torch.cuda.synchronize(self.dev)
                self.last_block = {"phases": _lib.phase_ms(self.runner.ctx.handle),
                                   "leaf": _lib.level_info(self.runner.ctx.handle, self.levels)}
        else:
            nsec, rp, R0, nlog = 0, 32, np.zeros(0, np.int32), np.zeros(0, np.int32)
        # metadata exchange: common capacity, per-section sizes
        meta = torch.zeros(1 + 2 * maxn, dtype=torch.int32, device=self.dev)
        meta[0] = rp
        if nsec:
            meta[1:1 + nsec] = torch.from_numpy(R0).to(self.dev)
            meta[1 + maxn:1 + maxn + nsec] = torch.from_numpy(nlog).to(self.dev)
        metas = [torch.empty_like(meta) for _ in range(self.world)]
        self._all_gather(metas, meta)
        allm = torch.stack(metas).cpu().numpy()
        rpc = int(allm[:, 0].max())
        pbytes = self.runner.pack_bytes(rpc, se)
        pack = self._buf("pack", maxn * pbytes, torch.uint8)
        if nsec:
            self.runner.export(rpc, pack.data_ptr(), stream)
        # the one data-path collective: section states -> rank 0
        gl = [self._buf(f"g{r}", maxn * pbytes, torch.uint8) for r in range(self.world)] if self.rank == 0 else None
        self.torch.cuda.synchronize(self.dev)  # the export ran on the library's stream
        self._gather(pack, gl)
        logs = self._gather_logs() if gather_logs else None
        if self.rank == 0:
            allp = self._buf("allpack", S * pbytes, torch.uint8)
            R0a, nloga, k = [], [], 0
            for r in range(self.world):
                n = per[r]
                if n:
                    allp[k * pbytes:(k + n) * pbytes].copy_(gl[r][:n * pbytes])
                    R0a.extend(allm[r, 1:1 + n])
                    nloga.extend(allm[r, 1 + maxn:1 + maxn + n])
                    k += n
            self.runner.run_upper(allp.data_ptr(), self.top, rpc, np.array(R0a, np.int32),
                                  np.array(nloga, np.int32), stream)
        return logs

    def _gather_logs(self):
        """Each rank's section table + compact device log -> rank 0 (NCCL)."""
        torch, dist = self.torch, self.dist
        stream = torch.cuda.current_stream(self.dev).cuda_stream
        if self.block is not None:
            info, secs = self.runner.sections()
            n = int(info.n_records)
        else:
            secs, n = np.zeros((0, 5), np.int64), 0
        sizes = torch.tensor([n, secs.shape[0]], dtype=torch.int64, device=self.dev)
        alls = [torch.empty_like(sizes) for _ in range(self.world)]
        self._all_gather(alls, sizes)
        alls = torch.stack(alls).cpu().numpy()
        nmax, smax = int(alls[:, 0].max()), int(alls[:, 1].max())
        a = self._buf("la", nmax, torch.int32)
        b = self._buf("lb", nmax, torch.int32)
        d = self._buf("ld", nmax, torch.float64)
        k = self._buf("lk", nmax, torch.uint8)
        st = self._buf("ls", 5 * max(smax, 1), torch.int64)
        if n:
            self.runner.log_device(a.data_ptr(), b.data_ptr(), d.data_ptr(), k.data_ptr(), stream)
        if secs.shape[0]:
            st[:secs.size].copy_(torch.from_numpy(secs.reshape(-1)).to(self.dev))
        out = []
        for name, t in (("a", a), ("b", b), ("d", d), ("k", k), ("s", st)):
            g = [torch.empty_like(t) for _ in range(self.world)] if self.rank == 0 else None
            self._gather(t.contiguous(), g)
            out.append(g)
        if self.rank != 0:
            return None
        parts = []
        for r in range(self.world):
            nr, sr = int(alls[r, 0]), int(alls[r, 1])
            sec = out[4][r][:5 * sr].view(sr, 5).cpu().numpy() if sr else np.zeros((0, 5), np.int64)
            parts.append((sec.tolist(), out[0][r][:nr].cpu().numpy(), out[1][r][:nr].cpu().numpy(),
                          out[2][r][:nr].cpu().numpy(), out[3][r][:nr].cpu().numpy()))
        return parts

    def result(self, parts):
        """Rank 0: full RhsegResult = gathered lower-level logs + the upper
        levels run here (logs in canonical order)."""
        from .recursive import RecordList, collect_result, result_info
        from .sections import SectionId

        res = collect_result(self.runner.ctx, result_info(self.runner.ctx), self.edge, self.bands, self.levels)
        if parts is None:
            return res
        own = [(s.level, s.row, s.col, r) for s, r in res.section_logs]
        pieces = list(parts)
        flat = [(lv, rw, cl, 0, 0) for lv, rw, cl, _ in own]
        # upper levels (this ctx) as one more part
        a = np.concatenate([r.arrays()[0] for *_, r in own]) if own else np.zeros(0, np.int32)
        b = np.concatenate([r.arrays()[1] for *_, r in own]) if own else np.zeros(0, np.int32)
        d = np.concatenate([r.arrays()[2] for *_, r in own]) if own else np.zeros(0)
        k = np.concatenate([r.arrays()[3] for *_, r in own]) if own else np.zeros(0, np.uint8)
        off = 0
        for i, (lv, rw, cl, r) in enumerate(own):
            flat[i] = (lv, rw, cl, off, len(r))
            off += len(r)
        pieces.append((flat, a, b, d, k))
        ids, A, B, D, K = assemble_logs(self.levels, pieces)
        logs, o = [], 0
        for (lev, row, col), cnt in ids:
            logs.append((SectionId(lev, row, col), RecordList(A[o:o + cnt], B[o:o + cnt], D[o:o + cnt],
                                                            K[o:o + cnt])))
            o += cnt
        res.section_logs = logs
        return res


# ---------------------------------------------------------------------------
# bench leg (N > 1 under torchrun)
# ---------------------------------------------------------------------------
def bench_sharded(args, bm):
    """N > 1 leg of bench.py (launched by torchrun, one rank per GPU). `bm` is the
    bench module (workload table, config dict, clock sampler, CPU leg, roofline model);
    the package never imports the top-level script itself."""
    import ctypes
    import os
    import time

    import torch
    import torch.distributed as dist

    from .recursive import HsegParams, RhsegParams
    from .synth import gen_synthetic

    WORKLOADS, make_cube, cube_shape, ClockSampler = bm.WORKLOADS, bm.make_cube, bm.cube_shape, bm.ClockSampler

    # one process per GPU; RHSEG_DIST_BACKEND=gloo lets several ranks share one GPU
    # (the single-GPU test box) -- collectives then stage through host memory
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    backend = os.environ.get("RHSEG_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()
    name = args.workload
    spec, crop, levels, w, t, st = WORKLOADS[name]
    bands, edge, _ = cube_shape(name)
    dev = torch.device("cuda", local)
    top, blocks = shard_plan(levels, world)
    blk = blocks[rank]
    # this rank's image rows only (host memory and H2D scale with 1/world)
    et = edge >> (top - 1)
    r0, r1 = (blk[0] * et, (blk[0] + blk[2]) * et) if blk is not None else (0, 0)
    host = torch.empty((bands, max(r1 - r0, 1), edge), dtype=torch.float32, pin_memory=True)
    if r1 > r0:
        if crop is None:
            gen_synthetic(*spec, out=host.numpy(), rows=(r0, r1))
        else:
            host.numpy()[...] = make_cube(name)[:, r0:r1, :]
    cube = torch.empty((bands, edge, edge), dtype=torch.float32, device=dev)

    def upload():
        if r1 > r0:
            cube[:, r0:r1, :].copy_(host[:, :r1 - r0, :], non_blocking=True)

    upload()
    params = RhsegParams(HsegParams(w, t, bm.MEASURE_OF.get(name, "sqrt-bsmse")), levels, st)
    sh = ShardedRhseg(params, edge, bands, local)
    sh.record = True
    flush = torch.empty(2 * 126 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    for _ in range(args.warmup):
        sh.step(cube)
    torch.cuda.synchronize()
    times, launches = [], 0
    phases = np.zeros(4)
    n = ctypes.c_int64()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sh.step(cube, gather_logs=False)  # (the log gather is part of the e2e leg below)
            e1.record()
            torch.cuda.synchronize()
            dist.barrier()
            times.append(e0.elapsed_time(e1))
            sh.runner.lib.rhseg_result_launches(sh.runner.ctx.handle, ctypes.byref(n))
            launches += int(n.value)
            if sh.block is not None:
                phases += sh.last_block["phases"]
    phases /= max(1, args.steps)
    sh.record = False
    # end to end: this rank's rows H2D, the sharded run, logs gathered to rank 0,
    # root labels D2H on rank 0 (wall clock, max over ranks)
    lab = np.empty(edge * edge, np.int32)
    e2e = []
    for _ in range(max(1, args.steps)):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        upload()
        torch.cuda.synchronize()
        parts = sh.step(cube, gather_logs=True)
        if rank == 0:
            from . import _lib

            _lib.check(sh.runner.lib.rhseg_result_labels(sh.runner.ctx.handle, _lib.ptr(lab), None), "labels")
        torch.cuda.synchronize()
        e2e.append(time.perf_counter() - t0)
        del parts
    vals = torch.tensor([float(np.mean(times)), float(np.median(e2e)) * 1e3, float(launches), *phases.tolist()],
                        device=dev)
    mx = vals.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(vals, op=dist.ReduceOp.SUM)
    ms, e2e_ms, launches_total = float(mx[0]), float(mx[1]), int(vals[2].item())
    ph_max = mx[3:7].cpu().numpy()  # per-kernel device ms of the slowest rank
    if rank == 0:
        npxb = edge * edge * bands
        leaf = sh.last_block["leaf"] if sh.block is not None else None
        roof = roof2 = None
        if leaf is not None:
            # the slowest rank's loop time against the whole job's algorithmic work
            roof, roof2 = bm.roofline(name, edge, bands, levels, w, ph_max, sh.runner.ctx.handle, leaf=leaf)
        line = {
            "metric": "RHSEG pixel-bands/sec", "value": npxb / (ms * 1e-3), "unit": "pixel-bands/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gen_synthetic, bit-identical to the reference generator)",
            "config": bm.config_of(name),
            "execution": f"subtree sharding: level-{top} subtrees over {world} ranks (no data-path collective "
                         f"below level {top}), NCCL gather of the level-{top} section states to rank 0, which "
                         f"runs the levels above",
            "phase_ms_max_over_ranks": {"init_stitch": float(ph_max[0]), "dinit_allpairs": float(ph_max[1]),
                                        "merge_loop": float(ph_max[2]), "resolve_labels": float(ph_max[3])},
            "gpu_launches": launches_total,
            "roofline": roof,
            "roofline_secondary": roof2,
            "e2e": {"value": npxb / (e2e_ms * 1e-3), "unit": "pixel-bands/s",
                    "h2d_bytes_per_step": npxb * 4, "d2h_bytes_per_step": edge * edge * 4,
                    "ms_per_step": e2e_ms,
                    "note": "each rank uploads its own rows; merge logs gathered to rank 0 over NCCL"},
            "clocks": clk.summary(),
        }
        if not getattr(args, "no_cpu_baseline", False):
            cb = bm.cpu_sample(name, make_cube(name), seconds_hint=args.ref_seconds)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0
