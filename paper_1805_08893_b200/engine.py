"""Device-side driver of the geometry stage: owns the HBM-resident buffers and calls the
C ABI (include/vrgeom.h) on the current CUDA stream.  PyTorch is used for device memory,
streams and torch.distributed only.

Layout in HBM:
  indices        uint32[I]            (held as an int32 tensor, same bits)
  positions4     float32[V,4]         (x, y, z, 1) -- one 16-byte gather per invocation
  offsets        int32[n_batches+1]   the "auxiliary buffer" (batching.py:128-137)
  unique_ids     uint32[N_inv]        per-round unique ids, concatenated in batch order
  assembly_map   uint16[I]            local index of every consumed slot
  shaded4        float32[N_inv,4]     (x/w, y/w, z/w, w)
  round tables   int32                batch_round_off, round_uid_off, round_prims
  stats          int64[16]
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .batching import BatchConfig, ConfigError, UnsupportedOnDevice


def _device(device=None) -> torch.device:
    N.require_cuda()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream_ptr():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _cfg_c(cfg: BatchConfig) -> N.BatchConfigC:
    return N.BatchConfigC(cfg.batch_size, cfg.max_unique, cfg.max_indices, cfg.warp_width,
                          cfg.block_size, cfg.primitive_size)


def _hash_c(hcfg) -> N.HashConfigC:
    return N.HashConfigC(hcfg.table_size, hcfg.multiplier, hcfg.max_fast_probes)


def raise_status(status: int, batch: int = -1):
    """Map a vr_status to the exception type the reference raises for the same condition."""
    if status == N.VR_OK:
        return
    msg = N.status_string(status) + (f" (batch {batch})" if batch >= 0 else "")
    if status in (N.VR_ERR_HASH_FULL, N.VR_ERR_WARP_NO_PROGRESS):
        raise RuntimeError(msg)  # strategies.py:283-284, :226-227
    if status == N.VR_ERR_UNSUPPORTED:
        raise UnsupportedOnDevice(msg)
    if status == N.VR_ERR_CUDA:
        raise N.NativeLibraryError(msg)
    if status in (N.VR_ERR_CAPACITY, N.VR_ERR_WORKSPACE):
        raise RuntimeError(msg)
    if status == N.VR_ERR_VERTEX_RANGE:
        raise IndexError(msg)  # strategies.py:62-65 positions[vid]
    raise ConfigError(msg)


def to_device_indices(indices, device=None) -> torch.Tensor:
    """uint32 index buffer -> int32 CUDA tensor with the same bits (borrowed if already there)."""
    dev = _device(device)
    if isinstance(indices, torch.Tensor):
        t = indices
        if t.dtype == torch.uint32:
            t = t.view(torch.int32)
        if t.dtype != torch.int32:
            t = t.to(torch.int64).to(torch.int32)
        return t.to(dev).contiguous()
    arr = np.ascontiguousarray(np.asarray(indices), dtype=np.uint32)
    return torch.from_numpy(arr.view(np.int32).copy()).to(dev)


def to_device_positions4(positions, device=None) -> torch.Tensor:
    """(V,3) float64/float32 -> float32[V,4] = (x,y,z,1) on the device (16-byte records)."""
    dev = _device(device)
    if isinstance(positions, torch.Tensor):
        p = positions.to(dev, torch.float32)
    else:
        p = torch.from_numpy(np.ascontiguousarray(positions, dtype=np.float32)).to(dev)
    out = torch.ones((p.shape[0], 4), dtype=torch.float32, device=dev)
    out[:, :3] = p
    return out


def static_offsets_device(index_count: int, cfg: BatchConfig, device=None) -> torch.Tensor:
    """batching.py:76-84 as a device-resident int32 offsets array (vr_static_offsets)."""
    lib = N.require_cuda()
    dev = _device(device)
    if index_count % cfg.primitive_size != 0:
        raise ConfigError(f"index count {index_count} is not primitive-aligned")
    c = _cfg_c(cfg)
    nb = lib.vr_static_batch_count(index_count, C.byref(c))
    if nb == 0:
        return torch.zeros(0, dtype=torch.int32, device=dev)
    offs = torch.empty(nb + 1, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        raise_status(lib.vr_static_offsets(index_count, C.byref(c), _ptr(offs), _stream_ptr()))
    offs.vr_static_batch_size = cfg.batch_size  # lets the runner pick the position-aligned kernels
    return offs


def dynamic_offsets_device(indices, cfg: BatchConfig, device=None, workspace=None, sync: bool = True):
    """batching.py:87-125 on the GPU -> int32 offsets (length n_batches+1; length 0 if empty).

    sync=False: no host round trip -- returns (offsets at full capacity, counts) where counts is the device int64[2]
    {batch count, vr_status} of vr_dynamic_batches; hand both to run_device(..., counted=(offsets, counts)), which
    launches for the upper bound vr_dynamic_batch_bound and lets the kernels read the count (vr_run_counted)."""
    lib = N.require_cuda()
    d_idx = to_device_indices(indices, device)
    dev = d_idx.device
    n = d_idx.numel()
    ps = cfg.primitive_size
    if n % ps != 0:
        raise ConfigError(f"index count {n} is not primitive-aligned")
    if n == 0:
        return torch.zeros(0, dtype=torch.int32, device=dev)
    c = _cfg_c(cfg)
    ws_bytes = lib.vr_dynamic_workspace_bytes(n, C.byref(c))
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    offs = torch.empty(n // ps + 1, dtype=torch.int32, device=dev)
    nb = torch.zeros(2, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        raise_status(lib.vr_dynamic_batches(_ptr(d_idx), n, C.byref(c), _ptr(offs), _ptr(nb),
                                            _ptr(workspace), ws_bytes, _stream_ptr()))
    if not sync:
        return offs, nb
    nbh = nb.cpu()
    if int(nbh[1]) != 0:
        raise_status(int(nbh[1]))
    return offs[: int(nbh[0]) + 1]


@dataclass
class ShaderSpec:
    """Closed set of device shaders (strategies.py:36-67)."""

    kind: int = N.VR_SHADER_NONE
    positions4: torch.Tensor | None = None
    matrix: np.ndarray | None = None
    attributes: torch.Tensor | None = None  # int32[V, words]
    vertex_count: int = 0
    batch_vertex_base: torch.Tensor | None = None  # int32[n_batches]: multi-draw (draws.py)
    extra_cycles: int = 0  # synthetic shader load per invocation (ShaderFn.cycles - 1)


class DeviceRun:
    """Result of one strategy run, resident on the device (flattened DedupResult list)."""

    def __init__(self):
        self.strategy = ""
        self.primitive_size = 3
        self.n_batches = 0
        self.batch_begin = self.batch_end = None
        self.batch_round_off = self.round_uid_off = self.round_prims = None
        self.unique_ids = self.assembly_map = self.shaded4 = self.shaded_attr = None
        self.shade_counts = None
        self.stats_dev = None
        self.launches = 0
        self.kernel_path = 0
        self.stream_xyz = None  # the output queue, when the run was asked for it (want_queue)
        self._counted = False   # launched through vr_run_counted: n_batches is an upper bound until the statistics are read
        self._stats = None

    def relaunch(self) -> "DeviceRun":
        """Issue vr_run with the prepared arguments on the current stream (see run_device)."""
        lib = N.require_cuda()
        if self.shade_counts is not None:
            self.shade_counts.zero_()
        with torch.cuda.device(self._device):
            st = (lib.vr_run_counted if self._counted else lib.vr_run)(*self._args, _stream_ptr())
        raise_status(st)
        self._stats = None
        self.launches = lib.vr_last_launch_count()  # kernels this call launched (bench.py's gpu_launches)
        self.kernel_path = lib.vr_last_kernel_path()  # 3 = persistent tile kernel (include/vrgeom.h)
        return self

    # -- statistics -----------------------------------------------------------------
    def stats(self) -> np.ndarray:
        if self._stats is None:
            self._stats = self.stats_dev.cpu().numpy()
        return self._stats

    def check(self):
        """Raise what the reference would have raised for the first failing batch."""
        if self._counted:  # the true batch count arrives with the statistics block
            self.n_batches = int(self.stats()[N.VR_STAT_BATCHES])
        err = int(self.stats()[N.VR_STAT_ERROR])
        if err != -1:
            raise_status(err & 0xFF, err >> 8)
        return self

    @property
    def indices(self) -> int:
        return int(self.stats()[N.VR_STAT_INDICES])

    @property
    def invocations(self) -> int:
        return int(self.stats()[N.VR_STAT_INVOCATIONS])

    @property
    def rounds(self) -> int:
        return int(self.stats()[N.VR_STAT_ROUNDS])

    @property
    def probes(self):
        s = self.stats()
        return int(s[N.VR_STAT_PROBES_FAST]), int(s[N.VR_STAT_PROBES_SLOW]), int(s[N.VR_STAT_PROBE_MAX_CHAIN])

    # -- host views -------------------------------------------------------------------
    def flat(self) -> dict:
        """Host copies trimmed to the exact result sizes (numpy)."""
        self.check()
        r, u, m = self.rounds, self.invocations, self.indices
        out = {
            "batch_round_off": self.batch_round_off[: self.n_batches + 1].cpu().numpy().astype(np.int64),
            "round_uid_off": self.round_uid_off[: r + 1].cpu().numpy().astype(np.int64),
            "round_prims": self.round_prims[:r].cpu().numpy(),
            "unique_ids": self.unique_ids[:u].cpu().numpy().view(np.uint32),
            "assembly_map": self.assembly_map[:m].cpu().numpy().view(np.uint16).astype(np.int32),
        }
        if self.n_batches == 0:
            out["batch_round_off"] = np.zeros(1, dtype=np.int64)
            out["round_uid_off"] = np.zeros(1, dtype=np.int64)
        if self.shaded4 is not None:
            out["shaded"] = self.shaded4[:u].cpu().numpy()
        if self.shaded_attr is not None:
            out["shaded_attr"] = self.shaded_attr[:u].cpu().numpy()
        if self.shade_counts is not None:
            out["shade_counts"] = self.shade_counts.cpu().numpy().astype(np.int64)
        return out

    def shaded_xyz(self, count: int | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
        """The shaded records in the reference's layout, float32[count, 3] (strategies.py:53-67), packed on the device
        (vr_pack_xyz): what crosses PCIe when the host wants the records."""
        lib = N.require_cuda()
        n = self.invocations if count is None else count
        if out is None:
            out = torch.empty((n, 3), dtype=torch.float32, device=self.stats_dev.device)
        with torch.cuda.device(self.stats_dev.device):
            raise_status(lib.vr_pack_xyz(_ptr(self.shaded4), n, _ptr(out), _stream_ptr()))
        return out[:n]

    def assembly_map_u8(self, count: int | None = None, out: torch.Tensor | None = None, flag: torch.Tensor | None = None):
        """The local indices as bytes (vr_pack_bytes): they are < warp_width resp. <= max_unique <= 256 in every configuration
        of the paper, and half as many bytes cross PCIe.  `flag` (int32[1], zeroed by the caller) is set if one did not fit."""
        lib = N.require_cuda()
        n = self.indices if count is None else count
        if out is None:
            out = torch.empty(n + 16, dtype=torch.uint8, device=self.stats_dev.device)
        with torch.cuda.device(self.stats_dev.device):
            raise_status(lib.vr_pack_bytes(_ptr(self.assembly_map), n, _ptr(out), _ptr(flag) if flag is not None else None,
                                        _stream_ptr()))
        return out[:n]

    def expand_stream(self, positions: bool):
        """Per-corner record stream (strategies.py:456-463) built on the device."""
        self.check()
        lib = N.require_cuda()
        m = self.indices
        dev = self.stats_dev.device
        if positions and self.stream_xyz is not None:  # written by the stage itself
            return self.stream_xyz[: 3 * m].view(m, 3)
        if positions:
            out = torch.empty((m, 3), dtype=torch.float32, device=dev)
        else:
            out = torch.empty(m, dtype=torch.int32, device=dev)
        if m == 0:
            return out
        ws = torch.empty((self.n_batches + 1) * 4 + 256, dtype=torch.uint8, device=dev)
        with torch.cuda.device(dev):
            raise_status(lib.vr_expand_stream(
                _ptr(self.batch_round_off), _ptr(self.round_uid_off), _ptr(self.round_prims),
                _ptr(self.assembly_map), _ptr(self.unique_ids), _ptr(self.shaded4) if positions else None,
                self.n_batches, _ptr(self.batch_begin), _ptr(self.batch_end), self.primitive_size,
                _ptr(out) if positions else None, None if positions else _ptr(out),
                _ptr(ws), ws.numel(), _stream_ptr()))
        return out


def ideal_counts(d_indices: torch.Tensor, vertex_count: int):
    """analytics.py:105-119 on the device: (number of referenced vertices, int32[vertex_count] 0/1 flags)."""
    lib = N.require_cuda()
    dev = d_indices.device
    counts = torch.empty(max(vertex_count, 1), dtype=torch.int32, device=dev)
    out = torch.zeros(2, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        raise_status(lib.vr_ideal_counts(_ptr(d_indices), d_indices.numel(), vertex_count, _ptr(counts), _ptr(out),
                                         _stream_ptr()))
    referenced, status = (int(v) for v in out.cpu().numpy())
    if status:
        raise_status(status)
    return referenced, counts[:vertex_count]


class RunBuffers:
    """Reusable output + workspace allocation for repeated runs of one shape (bench, serving)."""

    def __init__(self):
        self.t = {}

    def get(self, name, numel, dtype, device, zero=False):
        cur = self.t.get(name)
        if cur is None or cur.numel() < numel or cur.dtype != dtype or cur.device != device:
            cur = torch.empty(max(int(numel), 1), dtype=dtype, device=device)
            self.t[name] = cur
        if zero:
            cur.zero_()
        return cur


def run_device(strategy: str, d_indices: torch.Tensor, d_begin: torch.Tensor, d_end: torch.Tensor,
               n_batches: int, span_total: int, max_span: int, cfg: BatchConfig, hcfg=None,
               shader: ShaderSpec | None = None, *, want_counts: bool = False,
               buffers: RunBuffers | None = None, enforce_budget: bool = True,
               contiguous: bool | None = None, static: bool = False, fuse: bool = True,
               want_queue: bool = False, counted=None, plan_only: bool = False) -> DeviceRun:
    """vr_run on the current stream.  No host synchronisation; call .check()/.flat() to read back.
    `plan_only` prepares buffers and arguments without launching: `.relaunch()` then issues the same
    run again (same inputs, outputs overwritten) at the cost of one C call, for callers that repeat a
    run of one shape (a frame loop, bench.py)."""
    lib = N.require_cuda()
    if strategy not in N.STRATEGY_IDS:
        raise ConfigError(f"unknown strategy {strategy!r}; expected one of {tuple(N.STRATEGY_IDS)}")
    sid = N.STRATEGY_IDS[strategy]
    dev = d_indices.device
    if counted is not None:
        # (offsets at full capacity, device batch count) straight from dynamic_offsets_device(sync=False): sized for the
        # upper bound, the kernels read the count (vr_run_counted); d_begin / d_end / n_batches / span_total are derived
        c_offs, c_counts = counted
        n_batches = int(lib.vr_dynamic_batch_bound(d_indices.numel(), C.byref(_cfg_c(cfg)), 0))
        n_batches = min(n_batches, int(c_offs.numel()) - 1)
        d_begin, d_end, span_total, contiguous = c_offs[:-1], c_offs[1:], int(d_indices.numel()), True
    if contiguous is None:  # begin/end are two views of one offsets array
        contiguous = (n_batches > 0 and d_begin.data_ptr() + 4 == d_end.data_ptr()
                      and d_begin.is_contiguous() and d_end.is_contiguous())
    flags = ((0 if enforce_budget else N.VR_FLAG_NO_BUDGET) | (N.VR_FLAG_CONTIGUOUS if contiguous else 0)
             | (N.VR_FLAG_STATIC if static else 0) | (0 if fuse else N.VR_FLAG_NO_FUSE))
    shader = shader or ShaderSpec()
    buffers = buffers or RunBuffers()
    c = _cfg_c(cfg)
    h = _hash_c(hcfg) if hcfg is not None else None
    hp = C.byref(h) if h is not None else None
    max_inv, max_rounds = C.c_int64(0), C.c_int64(0)
    raise_status(lib.vr_output_bounds(sid, span_total, n_batches, C.byref(c), hp,
                                      C.byref(max_inv), C.byref(max_rounds)))
    ws_bytes = lib.vr_run_workspace_bytes(sid, span_total, n_batches, C.byref(c), hp)
    run = DeviceRun()
    run.strategy, run.primitive_size, run.n_batches = strategy, cfg.primitive_size, n_batches
    run.batch_begin, run.batch_end = d_begin, d_end
    g = buffers.get
    run.batch_round_off = g("bro", n_batches + 1, torch.int32, dev)
    run.round_uid_off = g("ruo", max_rounds.value + 1, torch.int32, dev)
    run.round_prims = g("rp", max_rounds.value, torch.int32, dev)
    run.unique_ids = g("uid", max_inv.value, torch.int32, dev)
    run.assembly_map = g("amap", span_total + 8, torch.int16, dev)
    run.stats_dev = g("stats", N.VR_STATS_WORDS, torch.int64, dev)
    ws = g("ws", ws_bytes + 256, torch.uint8, dev)
    sh = N.ShaderC()
    sh.kind = shader.kind
    sh.vertex_count = shader.vertex_count
    sh.extra_cycles = int(shader.extra_cycles)
    if shader.batch_vertex_base is not None:
        sh.d_batch_vertex_base = shader.batch_vertex_base.data_ptr()
    if shader.kind == N.VR_SHADER_POSITION:
        run.shaded4 = g("shaded", max_inv.value * 4, torch.float32, dev).view(-1, 4)
        sh.d_positions4 = shader.positions4.data_ptr()
        if shader.matrix is not None:
            sh.has_matrix = 1
            sh.matrix = (C.c_float * 16)(*np.asarray(shader.matrix, dtype=np.float32).reshape(16))
    if shader.attributes is not None:
        words = int(shader.attributes.shape[1])
        sh.d_attributes = shader.attributes.data_ptr()
        sh.attr_words = words
        run.shaded_attr = g("sattr", max_inv.value * words, torch.int32, dev).view(-1, words)
    if want_queue:  # the stage's output queue: one float32[3] record per corner (vr_outputs.d_stream_xyz)
        if shader.kind != N.VR_SHADER_POSITION:
            raise ConfigError("the output queue holds shaded positions: position shader only")
        run.stream_xyz = g("queue", span_total * 3 + 16, torch.float32, dev)
    if want_counts:
        if shader.vertex_count <= 0:
            raise ConfigError("per-vertex tallies need vertex_count")
        run.shade_counts = g("counts", shader.vertex_count, torch.int32, dev, zero=True)
    out = N.OutputsC(
        run.batch_round_off.data_ptr(), run.round_uid_off.data_ptr(), run.round_prims.data_ptr(),
        run.unique_ids.data_ptr(), run.assembly_map.data_ptr(),
        run.shaded4.data_ptr() if run.shaded4 is not None else None,
        run.shaded_attr.data_ptr() if run.shaded_attr is not None else None,
        run.shade_counts.data_ptr() if run.shade_counts is not None else None,
        run.stats_dev.data_ptr(), max_inv.value, max_rounds.value,
        run.stream_xyz.data_ptr() if run.stream_xyz is not None else None)
    if counted is not None:
        args = (sid | flags, _ptr(d_indices), d_indices.numel(), _ptr(counted[0]), n_batches, _ptr(counted[1]), max_span,
                C.byref(c), hp, C.byref(sh), C.byref(out), _ptr(ws), ws.numel())
        run._counted = True
    else:
        args = (sid | flags, _ptr(d_indices), d_indices.numel(), _ptr(d_begin), _ptr(d_end), n_batches,
                span_total, max_span, C.byref(c), hp, C.byref(sh), C.byref(out), _ptr(ws), ws.numel())
    run._keep = (ws, shader, c, h, sh, out, d_indices, d_begin, d_end, counted)
    run._args, run._device = args, dev
    if plan_only:
        return run
    return run.relaunch()
