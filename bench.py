#!/usr/bin/env python
"""bench.py -- Stream VByte on B200: the BASELINE.json metric on its configs.

Workloads (BASELINE.json configs; seeded synthetic inputs):
  cfg2  delta encode + decode of one sorted 2^26-uint32 array (gaps mean 8), prev = 0
  cfg3  plain encode + decode of one 2^28-uint32 array, byte length uniform 1..4
        (the largest single-GPU single-array config: the N=1 headline)
  cfg4  1M posting-list-like arrays (~2^30 integers), per-list delta, batch kernels
  cfg5  2^31 sorted integers in 64K-integer prev-seeded chunks, delta, batch kernels

A step is one round trip of the workload -- the encode call and the decode call,
each CUDA-event timed on its launch stream with inputs resident in HBM and L2
flushed before it.  `value` = integers round-tripped per second over all ranks.

  python bench.py                      N=1: headline cfg3, cfg2/cfg4/cfg5 under "workloads"
  python bench.py --gpus N             N>1: spawns N ranks (torch.distributed.run) unless
                                       launched by one; cfg5 chunks (or --workload cfg4
                                       lists) sharded across ranks, no collective on the
                                       data path; the gather to rank 0 is timed separately
  python bench.py --impl reference     the CPU reference (the pinned oracle port: the
                                       reference itself is headers-only) on the same
                                       workload and n, all host threads; loads no codec .so

JSON line keys follow the driver contract (see DESIGN.md §4 for each key).
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "billions of uint32/sec decoded (plain & delta) and encoded; % of HBM roofline"
WORKLOADS = ("cfg2", "cfg3", "cfg4", "cfg5")
DECODE_SEG_DTYPE = np.dtype([("src_offset", "<u8"), ("src_bytes", "<u8"), ("dst_offset", "<u8"),
                             ("n", "<u4"), ("prev", "<u4")])
ENCODE_SEG_DTYPE = np.dtype([("src_offset", "<u8"), ("dst_capacity", "<u8"), ("dst_offset", "<u8"),
                             ("n", "<u4"), ("prev", "<u4")])


def _gen():
    """The synthetic-input generator, loaded as a standalone file: it maps only
    libsvbgen.so, so the reference arm never loads the codec library."""
    mod = sys.modules.get("svb_gen_standalone")
    if mod is None:
        spec = importlib.util.spec_from_file_location("svb_gen_standalone", ROOT / "paper_1709_08990_b200" / "gen.py")
        mod = importlib.util.module_from_spec(spec)
        sys.modules["svb_gen_standalone"] = mod
        spec.loader.exec_module(mod)
    return mod


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# clocks sampling during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        t_wait = time.time()
        while self.proc and not self.lines and time.time() - t_wait < 3.0:
            time.sleep(0.02)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self._t:
                self._t.join(timeout=2)

    def summary(self, first: int = 0):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[max(0, first):]:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9 or f[0] != str(self.gpu):
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "window": "timed region + identical untimed load to 0.4 s (nvidia-smi -lms 100)"}


# ---------------------------------------------------------------------------
# workloads: host data of one rank (each rank generates only its own shard)
# ---------------------------------------------------------------------------
def _load_shard():
    """shard.partition_by_cost, loaded standalone (shard.py is numpy-only: no codec library)."""
    spec = importlib.util.spec_from_file_location("svb_shard_standalone", ROOT / "paper_1709_08990_b200" / "shard.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.partition_by_cost


_partition = _load_shard()


class SingleArray:
    """cfg2 / cfg3: one array (single-array look-back kernels).  Does not shard:
    N>1 runs N independent replicas."""
    batch = False

    def __init__(self, cfg: int, n: int | None = None):
        gen = _gen()
        self.cfg, self.delta = cfg, cfg == 2
        self.name = f"cfg{cfg}"
        self.values = gen.config_array(cfg, n)
        self.n = int(self.values.size)
        self.nseg = 1

    def describe(self):
        if self.cfg == 2:
            return {"workload": "cfg2", "what": "delta encode+decode of one sorted array, geometric gaps mean 8, prev=0",
                    "n": self.n}
        return {"workload": "cfg3", "what": "plain encode+decode of one array, byte length uniform 1-4", "n": self.n}

    # --- device (product) side ---
    def setup(self, dev, torch):
        self.dev = dev
        self.d_v = torch.from_numpy(self.values.view(np.int32)).cuda()
        cap = (self.n + 3) // 4 + 4 * self.n
        self.d_c = torch.empty(cap, dtype=torch.uint8, device="cuda")
        self.d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.d_o = torch.empty_like(self.d_v)
        self.d_last = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.encode()
        torch.cuda.synchronize()
        self.cmp = int(self.d_len.item())

    def encode(self):
        self.dev.encode(self.d_v, self.d_c, self.d_len, delta=self.delta, prev=0)

    def decode(self):
        self.dev.decode(self.d_c, self.n, self.d_o, in_len=self.cmp, delta=self.delta, base=0, last=self.d_last)

    def verify(self, torch):
        self.dev.check()
        assert torch.equal(self.d_o, self.d_v), "round trip mismatch"

    def release(self):
        for k in ("d_v", "d_c", "d_len", "d_o", "d_last", "h_v", "h_c", "h_o"):
            self.__dict__.pop(k, None)

    # --- e2e through the reference-facing host C-ABI (pinned host buffers) ---
    def e2e_setup(self, torch):
        self.h_v = torch.from_numpy(self.values.view(np.int32)).pin_memory()
        self.h_c = torch.empty((self.n + 3) // 4 + 4 * self.n, dtype=torch.uint8).pin_memory()
        self.h_o = torch.empty(self.n, dtype=torch.int32).pin_memory()

    def e2e_step(self):
        import ctypes as C

        from paper_1709_08990_b200 import codec
        from paper_1709_08990_b200._native import lib
        ctx = codec._ctx(int(os.environ.get("BENCH_DEVICE", "0")))
        ln = C.c_size_t(0)
        st = lib.bcgpu_svb_encode_host(ctx, self.h_v.data_ptr(), self.n, int(self.delta), 0, self.h_c.data_ptr(),
                                       self.h_c.numel(), C.byref(ln))
        assert st == 0, st
        last = C.c_uint32(0)
        st = lib.bcgpu_svb_decode_host(ctx, self.h_c.data_ptr(), ln.value, self.n, int(self.delta), 0,
                                       self.h_o.data_ptr(), C.byref(last))
        assert st == 0, st
        return 4 * self.n + ln.value, ln.value + 4 * self.n  # h2d, d2h bytes

    def e2e_verify(self):
        assert np.array_equal(self.h_o.numpy().view(np.uint32), self.values)

    e2e_path = "bcgpu_svb_encode_host + bcgpu_svb_decode_host (pinned host buffers, piecewise 3-stream pipeline)"


class Batch:
    """cfg4 / cfg5: independent segments (batch kernels), sharded across ranks by
    contiguous segment ranges of equal cost; rank r generates only its shard."""
    batch = True

    def __init__(self, cfg: int, rank: int = 0, world: int = 1, scale: float = 1.0):
        gen = _gen()
        self.cfg, self.delta = cfg, True
        self.name = f"cfg{cfg}"
        if cfg == 4:
            nl = max(1, int((1 << 20) * scale))
            lens_all, self.cap = gen.list_lengths(nl, gen.SEEDS[4], cap_total=int((1 << 30) * scale))
            # cost of a list ~ its algorithmic bytes: 4n + ~2.3n compressed
            lo, hi = _partition(lens_all.astype(np.float64) * 6.3, world)[rank]
            lb = gen.posting_lists_range(lens_all, lo, hi, gen.SEEDS[4])
            self.values, self.lens, self.offs = lb.values, lb.lengths, lb.offsets
            self.prevs = np.zeros(hi - lo, np.uint32)
        else:
            chunk = gen.CFG5_CHUNK
            nl = max(1, int((1 << 31) * scale) // chunk)
            lo, hi = _partition(np.ones(nl), world)[rank]
            i0, m = lo * chunk, (hi - lo) * chunk
            if i0:  # one extra element: the previous chunk's last value seeds this shard's first prev
                v = gen.geometric_sorted_range(i0 - 1, m + 1, 32.0, gen.SEEDS[5])
                first_prev, self.values = int(v[0]), v[1:]
            else:
                first_prev, self.values = 0, gen.geometric_sorted_range(0, m, 32.0, gen.SEEDS[5])
            self.lens = np.full(hi - lo, chunk, np.uint32)
            self.offs = np.arange(hi - lo + 1, dtype=np.uint64) * chunk
            self.prevs = np.zeros(hi - lo, np.uint32)
            if hi > lo:
                self.prevs[0] = first_prev
                self.prevs[1:] = self.values[chunk - 1:-1:chunk]
            self.cap = None
        self.seg_lo, self.seg_hi = lo, hi
        self.n = int(self.values.size)
        self.nseg = hi - lo
        self.max_n = int(self.lens.max()) if self.nseg else 0
        self.total_segments = int(nl)

    def describe(self):
        if self.cfg == 4:
            return {"workload": "cfg4", "what": "1M posting-list-like arrays, delta encode+decode per list (prev=0), "
                                                "water-fill capped to 2^30 ints", "lists": self.total_segments,
                    "cap": self.cap, "n": self.n}
        return {"workload": "cfg5", "what": "2^31 sorted ints (gaps mean 32, wrapping) in 64K-int chunks, "
                                            "prev-seeded delta encode+decode", "chunks": self.total_segments,
                "n": self.n}

    def host_segments(self):
        """Encode descriptors over worst-case slots (the device layout the timed calls use)."""
        caps = (self.lens.astype(np.uint64) + 3) // 4 + 4 * self.lens.astype(np.uint64)
        eoff = np.zeros(self.nseg + 1, np.uint64)
        np.cumsum(caps, out=eoff[1:])
        es = np.zeros(self.nseg, ENCODE_SEG_DTYPE)
        es["src_offset"], es["dst_capacity"], es["dst_offset"] = self.offs[:-1], caps, eoff[:-1]
        es["n"], es["prev"] = self.lens, self.prevs
        return es, eoff

    def setup(self, dev, torch):
        from paper_1709_08990_b200.device import segments_to_tensor
        self.dev = dev
        es, eoff = self.host_segments()
        self.eoff = eoff
        self.d_esegs = segments_to_tensor(es, "cuda")
        self.d_v = torch.from_numpy(self.values.view(np.int32)).cuda()
        self.d_c = torch.empty(int(eoff[-1]) + 16, dtype=torch.uint8, device="cuda")
        self.d_lens = torch.zeros(max(1, self.nseg), dtype=torch.int64, device="cuda")
        self.d_o = torch.empty_like(self.d_v)
        self.encode()
        torch.cuda.synchronize()
        lens = self.d_lens.cpu().numpy()[: self.nseg].astype(np.uint64)
        self.cmp = int(lens.sum())
        self.enc_lens = lens
        ds = np.zeros(self.nseg, DECODE_SEG_DTYPE)
        ds["src_offset"], ds["src_bytes"], ds["dst_offset"] = eoff[:-1], lens, self.offs[:-1]
        ds["n"], ds["prev"] = self.lens, self.prevs
        self.d_dsegs = segments_to_tensor(ds, "cuda")

    def encode(self):
        self.dev.encode_batch(self.d_esegs, self.nseg, self.d_v, self.d_c, self.d_lens, delta=True,
                              max_seg_n=self.max_n)

    def decode(self):
        self.dev.decode_batch(self.d_dsegs, self.nseg, self.d_c, self.d_o, delta=True, max_seg_n=self.max_n)

    def verify(self, torch):
        self.dev.check()
        assert torch.equal(self.d_o, self.d_v), "round trip mismatch"

    def release(self):
        for k in ("d_esegs", "d_v", "d_c", "d_lens", "d_o", "d_dsegs", "h_v", "h_c", "h_o"):
            self.__dict__.pop(k, None)

    # --- e2e through the host batch C-ABI (bcgpu_svb_{encode,decode}_batch_host) ---
    def e2e_setup(self, torch):
        self.h_v = torch.from_numpy(self.values.view(np.int32)).pin_memory()
        cap = int(((self.lens.astype(np.uint64) + 3) // 4 + 4 * self.lens.astype(np.uint64)).sum())
        self.h_c = torch.empty(max(1, cap), dtype=torch.uint8).pin_memory()
        self.h_o = torch.empty(max(1, self.n), dtype=torch.int32).pin_memory()
        self.h_lens = np.ascontiguousarray(self.lens, np.uint32)
        self.h_prevs = np.ascontiguousarray(self.prevs, np.uint32)
        self.h_offs = np.zeros(self.nseg + 1, np.uint64)

    def e2e_step(self):
        from paper_1709_08990_b200 import codec
        from paper_1709_08990_b200._native import lib
        ctx = codec._ctx(int(os.environ.get("BENCH_DEVICE", "0")))
        st = lib.bcgpu_svb_encode_batch_host(ctx, self.h_v.data_ptr(), self.h_lens.ctypes.data,
                                             self.h_prevs.ctypes.data, self.nseg, 1, self.h_c.data_ptr(),
                                             self.h_c.numel(), self.h_offs.ctypes.data)
        assert st == 0, st
        cmp = int(self.h_offs[-1])
        st = lib.bcgpu_svb_decode_batch_host(ctx, self.h_c.data_ptr(), cmp, self.h_offs.ctypes.data,
                                             self.h_lens.ctypes.data, self.h_prevs.ctypes.data, self.nseg, 1,
                                             self.h_o.data_ptr(), None)
        assert st == 0, st
        seg_bytes = 8 * self.nseg
        h2d = 4 * self.n + seg_bytes + cmp + 8 * (self.nseg + 1) + seg_bytes
        d2h = cmp + 8 * (self.nseg + 1) + 4 * self.n
        return h2d, d2h

    def e2e_verify(self):
        assert np.array_equal(self.h_o.numpy()[: self.n].view(np.uint32), self.values)
        assert int(self.h_offs[-1]) == self.cmp

    e2e_path = ("bcgpu_svb_encode_batch_host + bcgpu_svb_decode_batch_host (pinned host buffers; in-library "
                "size pass, packing scan and exact-size transfers, pipelined over pieces of segments)")


def make_workload(name: str, rank: int, world: int, n: int | None, scale: float):
    if name == "cfg2":
        return SingleArray(2, n)
    if name == "cfg3":
        return SingleArray(3, n)
    if name in ("cfg4", "cfg5"):
        return Batch(int(name[-1]), rank, world, scale)
    raise SystemExit(f"unknown workload {name}")


# ---------------------------------------------------------------------------
# CPU reference (the pinned oracle port; the reference itself is headers-only)
# ---------------------------------------------------------------------------
def _oracle():
    import oracle
    return oracle


def cpu_round_trip(wl, threads: int, n_sample: int | None, min_seconds: float, min_reps: int = 3):
    """All-core round trip of (a bounded sample of) the workload with the oracle port:
    O1 encoder + O2 (paper Fig. 4 SSSE3) decoder, pthreads over chunks / segments.
    Returns (per-rep Gint/s list, ints per rep, description)."""
    o = _oracle()
    bufs = wl.__dict__.setdefault("_cpu_bufs", {})  # reused across calls: no first-touch faults in the timing

    def buf(key, size, dtype):
        b = bufs.get(key)
        if b is None or b.size < size or b.dtype != dtype:
            b = bufs[key] = np.empty(size, dtype)
            b.fill(0)
        return b[:size]
    if not wl.batch:
        v = wl.values if not n_sample or n_sample >= wl.n else wl.values[:n_sample]
        out = buf("enc", (v.size + 3) // 4 + 4 * v.size + 1, np.uint8)
        dec = buf("dec", v.size, np.uint32)
        rates, t_total = [], 0.0
        while len(rates) < min_reps or t_total < min_seconds:
            t0 = time.perf_counter()
            m = o.mt_encode(v, delta=wl.delta, prev=0, threads=threads, out=out)
            st, _ = o.mt_decode(out[:m], v.size, dec, delta=wl.delta, base=0, threads=threads)
            dt = time.perf_counter() - t0
            t_total += dt
            rates.append(v.size / dt / 1e9)
            assert st == 0 and np.array_equal(dec, v)
        return rates, int(v.size), f"{v.size}-int {'prefix' if v.size < wl.n else 'whole array'} of the {wl.name} input"
    # batch: the first segments covering ~n_sample integers (every segment when n_sample is None)
    k = wl.nseg if not n_sample else int(np.searchsorted(wl.offs, n_sample, side="left"))
    k = max(1, min(k, wl.nseg))
    ni = int(wl.offs[k])
    es, eoff = wl.host_segments()
    es = es[:k]
    enc = buf("enc", int(eoff[k]) + 16, np.uint8)
    lens = np.zeros(k, np.uint64)
    dec = buf("dec", ni, np.uint32)
    ds = np.zeros(k, DECODE_SEG_DTYPE)
    ds["src_offset"], ds["dst_offset"], ds["n"], ds["prev"] = eoff[:k], wl.offs[:k], wl.lens[:k], wl.prevs[:k]
    vals = wl.values[:ni]
    rates, t_total = [], 0.0
    while len(rates) < min_reps or t_total < min_seconds:
        t0 = time.perf_counter()
        o.encode_batch(es, vals, enc, lens, True, threads)
        ds["src_bytes"] = lens
        st = o.decode_batch(ds, enc, dec, True, threads)
        dt = time.perf_counter() - t0
        t_total += dt
        rates.append(ni / dt / 1e9)
        assert st == 0 and np.array_equal(dec, vals)
    return rates, ni, f"first {k} of {wl.nseg} segments ({ni} ints) of the {wl.name} input"


def cpu_paper_mode(wl, n_sample: int, reps: int = 11):
    """The paper's methodology: ONE thread, O2 decode
    (delta included) from RAM into a reused 4096-integer buffer, median of >= 10 reps; plus
    the 1-thread O1 encode of the same sample.  Returns a dict of Gint/s figures."""
    o = _oracle()
    buf = np.empty(4096, np.uint32)
    if not wl.batch:
        v = wl.values[: min(n_sample, wl.n)]
        enc = np.frombuffer(o.encode(v, delta=wl.delta, prev=0), np.uint8)
        ni = v.size

        def dec_once():
            st, _ = o.paper_decode(enc, ni, wl.delta, 0, buf)
            assert st == 0
        out = np.empty(enc.size + 16, np.uint8)

        def enc_once():
            o.mt_encode(v, delta=wl.delta, prev=0, threads=1, out=out)
    else:
        k = max(1, min(wl.nseg, int(np.searchsorted(wl.offs, n_sample, side="left"))))
        ni = int(wl.offs[k])
        es, eoff = wl.host_segments()
        es = es[:k]
        encb = np.empty(int(eoff[k]) + 16, np.uint8)
        lens = np.zeros(k, np.uint64)
        o.encode_batch(es, wl.values[:ni], encb, lens, True, 1)
        ds = np.zeros(k, DECODE_SEG_DTYPE)
        ds["src_offset"], ds["src_bytes"], ds["dst_offset"] = eoff[:k], lens, wl.offs[:k]
        ds["n"], ds["prev"] = wl.lens[:k], wl.prevs[:k]

        def dec_once():
            st, _ = o.paper_decode_batch(ds, encb, True, buf)
            assert st == 0

        def enc_once():
            o.encode_batch(es, wl.values[:ni], encb, lens, True, 1)
    dec_once()
    d = []
    for _ in range(reps):
        t0 = time.perf_counter()
        dec_once()
        d.append(ni / (time.perf_counter() - t0) / 1e9)
    enc_once()
    e = []
    for _ in range(reps):
        t0 = time.perf_counter()
        enc_once()
        e.append(ni / (time.perf_counter() - t0) / 1e9)
    return {"decode_gint_s": round(statistics.median(d), 4), "decode_min": round(min(d), 4),
            "decode_max": round(max(d), 4), "encode_gint_s": round(statistics.median(e), 4),
            "encode_min": round(min(e), 4), "encode_max": round(max(e), 4), "reps": reps, "sample_ints": int(ni),
            "threads": 1,
            "mode": "O2 (paper Fig. 4 SSSE3) decode incl. delta, RAM -> reused 4096-int buffer (PAPER.md:415,436); "
                    "O1 encode RAM -> RAM; median of reps"}


def cpu_baseline(wl, args):
    threads = os.cpu_count() or 1
    rates, ni, what = cpu_round_trip(wl, threads, args.cpu_sample or (1 << 24), args.cpu_seconds)
    value = statistics.median(rates)
    res = {"value": round(value, 4), "unit": "Gint/s", "cores": threads, "kind": "port",
           "sample": f"{what}, encode+decode round trip, median of {len(rates)} reps (O1 encoder + SSSE3 Fig.4 "
                     f"decoder, {threads} pthreads over chunks/segments)",
           "min": round(min(rates), 4), "max": round(max(rates), 4), "cpu_model": _cpu_model(), "nproc": threads}
    if not args.no_paper_mode:
        res["paper_mode_1thread"] = cpu_paper_mode(wl, min(ni, 1 << 24))
    return res


def run_reference(args):
    """--impl reference: the CPU reference arm.  Rank 0 alone runs it (other ranks exit 0).
    Loads only the oracle and the standalone generator -- never libbytecodec_b200.so."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = args.gpus
    name = args.workload or ("cfg3" if world == 1 else "cfg5")
    wl = make_workload(name, 0, 1, args.n, args.scale)  # the whole job's workload (every rank's shard)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_round_trip(wl, threads, None, 0.0, min_reps=1)
    vals, t_all = [], time.perf_counter()
    for _ in range(args.steps):
        r, ni, what = cpu_round_trip(wl, threads, None, 0.0, min_reps=1)
        vals.append(r[0])
    elapsed = time.perf_counter() - t_all
    value = statistics.median(vals)
    sample = f"{what}, encode+decode round trip per step (the full workload, same n as the GPU arm)"
    loaded = _loaded_libs()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "Gint/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * elapsed / max(1, args.steps), 3),
        "higher_is_better": True, "scaling": "strong" if wl.batch else "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded splitmix64 generators standing in for BASELINE.json configs)",
        "config": dict(wl.describe(), same_config=True, threads=threads),
        "cpu_baseline": {"value": round(value, 4), "unit": "Gint/s", "cores": threads, "kind": "port",
                         "sample": sample, "cpu_model": _cpu_model()},
        "e2e": {"value": round(value, 4), "unit": "Gint/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_libs": loaded,
        "note": "the reference is headers-only (no src/*.cpp, SURVEY.md §0), so the CPU reference arm is the pinned "
                "oracle port: O1 encoder + paper Fig. 4 SSSE3 decoder, pthreads over chunks / segments",
    }
    print(json.dumps(line), flush=True)
    return 0


def _loaded_libs():
    try:
        return sorted({Path(ln.split()[-1]).name for ln in Path("/proc/self/maps").read_text().splitlines()
                       if ln.endswith(".so") and (str(ROOT) in ln or "/repo/" in ln)})
    except Exception:
        return []


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args) -> int:
    """--gpus N without a launcher: re-run this script under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd).returncode


class Dist:
    """Rank plumbing: NCCL when every rank has its own GPU, gloo when ranks share one."""

    def __init__(self, torch):
        self.torch = torch
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        ndev = max(1, torch.cuda.device_count())
        self.device = self.local % ndev
        self.shared_gpu = self.world > ndev
        torch.cuda.set_device(self.device)
        os.environ["BENCH_DEVICE"] = str(self.device)
        self.backend = None
        if self.world > 1:
            import torch.distributed as dist
            self.dist = dist
            self.backend = "gloo" if self.shared_gpu else "nccl"
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device))
            else:
                dist.init_process_group("gloo")

    def _t(self, x):
        t = self.torch.tensor([float(x)], dtype=self.torch.float64)
        return t.cuda() if self.backend == "nccl" else t

    def max(self, x: float) -> float:
        if self.world == 1:
            return float(x)
        t = self._t(x)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return float(x)
        t = self._t(x)
        self.dist.all_reduce(t)
        return float(t.item())

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def measure_workload(wl, dev, dst, args, torch, peak, peak_src):
    from paper_1709_08990_b200 import _native
    wl.setup(dev, torch)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    drain = torch.ones(64 << 20, dtype=torch.int32, device="cuda")

    def flush_l2(k):
        # evict L2: write 256 MiB, then read another 256 MiB so the dirty lines of the
        # write are written back here and not inside the next timed kernel
        flush.fill_(k)
        drain.sum()

    def step(evs):
        flush_l2(1)
        evs[0].record(stream)
        wl.encode()
        evs[1].record(stream)
        flush_l2(2)
        evs[2].record(stream)
        wl.decode()
        evs[3].record(stream)

    warm = max(3, args.warmup)
    for _ in range(warm):
        step([torch.cuda.Event(enable_timing=True) for _ in range(4)])
    torch.cuda.synchronize()
    wl.verify(torch)

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    clk = ClockSampler(dst.device).start()
    dst.barrier()
    torch.cuda.synchronize()
    first_sample = len(clk.lines)
    launches0 = _native.kernel_launch_count()
    t_timed = time.time()
    for k in range(args.steps):
        step(evs[k])
    torch.cuda.synchronize()
    launches = _native.kernel_launch_count() - launches0
    scratch = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    while time.time() - t_timed < 0.4:
        step(scratch)
        torch.cuda.synchronize()
    clk.stop()
    dst.barrier()
    t_enc = [e[0].elapsed_time(e[1]) for e in evs]
    t_dec = [e[2].elapsed_time(e[3]) for e in evs]
    me, md = statistics.mean(t_enc), statistics.mean(t_dec)
    ms_step = dst.max(statistics.mean(a + b for a, b in zip(t_enc, t_dec)))
    me_max, md_max = dst.max(me), dst.max(md)
    n_all = dst.sum(wl.n)
    alg_all = dst.sum(wl.cmp + 4 * wl.n)
    wl.verify(torch)

    # per-GPU roofline: the whole job's algorithmic bytes over the slowest rank's time, per GPU
    def phase(ms):
        gbs = alg_all / ms / 1e6
        return {"ms": round(ms, 4), "gint_s": round(n_all / ms / 1e6, 2), "gbs": round(gbs, 1),
                "frac": round(gbs / dst.world / peak, 4)}
    phases = {"encode": phase(me_max), "decode": phase(md_max)}
    dom = "decode" if md_max >= me_max else "encode"
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists() and dst.world == 1:
        traffic = json.loads(tf.read_text()).get(f"{wl.name}:{dom}")
    res = {
        "value": round(n_all / ms_step / 1e6, 3), "unit": "Gint/s", "ms_per_step": round(ms_step, 4),
        "config": dict(wl.describe(), n_all_ranks=int(n_all), compressed_bytes=int(dst.sum(wl.cmp)),
                       bytes_per_int=round(dst.sum(wl.cmp) / max(1.0, n_all), 4),
                       segments=int(dst.sum(wl.nseg)),
                       step="encode call + decode call (round trip), each CUDA-event timed on its stream",
                       l2="flushed before every timed call (256 MiB write, then a 256 MiB read that drains the "
                          "dirty lines)",
                       parallelism=(f"segment shards x{dst.world}" if wl.batch else f"replicas x{dst.world}")
                       + (" (ranks share one GPU: gloo)" if dst.shared_gpu else "")),
        "scaling": "strong" if wl.batch else "weak",
        "phases": phases,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(phases[dom]["gbs"] / dst.world, 1),
                     "peak": peak, "unit": "GB/s", "frac": phases[dom]["frac"], "traffic": traffic,
                     "algorithmic_bytes_per_launch": int(alg_all / dst.world),
                     "per_unit": f"{round((wl.cmp + 4 * wl.n) / max(1, wl.n), 4)} B per integer (cmp + 4n)",
                     "peak_source": peak_src},
        "gpu_launches": int(launches),
        "clocks": clk.summary(first_sample - 1),
    }
    # optional gather of the decoded shards to rank 0 (timed separately)
    if dst.world > 1 and wl.batch and not args.no_gather:
        res["gather"] = time_gather(wl, dst, torch)
    # e2e through the host C-ABI with pinned host buffers
    if not args.no_e2e:
        wl.e2e_setup(torch)
        wl.e2e_step()
        reps = max(3, min(args.steps, 5))
        dst.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            h2d, d2h = wl.e2e_step()
        torch.cuda.synchronize()
        t_e2e = dst.max((time.perf_counter() - t0) / reps)
        wl.e2e_verify()
        res["e2e"] = {"value": round(n_all / t_e2e / 1e9, 4), "unit": "Gint/s", "h2d_bytes_per_step": int(h2d),
                      "d2h_bytes_per_step": int(d2h), "ms_per_step": round(1e3 * t_e2e, 2), "path": wl.e2e_path}
    del flush, drain
    return res


def time_gather(wl, dst, torch):
    """Every rank's decoded shard to rank 0 (NCCL send/recv over NVLink; gloo via host when
    ranks share one GPU), timed on its own after the codec steps, max over ranks."""
    from paper_1709_08990_b200.shard import gather_to_root
    t = wl.d_o if dst.backend == "nccl" else wl.d_o.cpu()
    gather_to_root(t, dst.world, dst.rank)  # warm-up (connections, buffers)
    torch.cuda.synchronize()
    dst.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ev0.record()
    got = gather_to_root(t, dst.world, dst.rank)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) if dst.backend == "nccl" else 1e3 * (time.perf_counter() - t0)
    ms = dst.max(ms)
    total = dst.sum(4 * wl.n)
    ok = True
    if dst.rank == 0:
        ok = sum(int(x.numel()) for x in got) * 4 == int(total) and torch.equal(got[0].to(t.device), t)
    return {"ms": round(ms, 3), "bytes": int(total), "gbs": round(total / ms / 1e6, 1), "ok": bool(ok),
            "path": "torch.distributed send/recv to rank 0 (" + ("NCCL over NVLink/NVSwitch" if dst.backend == "nccl"
                                                               else "gloo through host memory") + ")",
            "timed": "separately, after the codec steps (not in value)"}


def run_gpu(args):
    import torch
    dst = Dist(torch)
    from paper_1709_08990_b200.device import DeviceCodec
    dev = DeviceCodec(dst.device)
    peak, peak_src = _peaks()
    if args.workload == "all" or args.workload is None:
        names = ["cfg3", "cfg2", "cfg4", "cfg5"] if dst.world == 1 else ["cfg5", "cfg4"]
        if args.workload is None and args.no_extra:
            names = names[:1]
    else:
        names = [args.workload]
    results = {}
    for name in names:
        wl = make_workload(name, dst.rank, dst.world, args.n, args.scale)
        r = measure_workload(wl, dev, dst, args, torch, peak, peak_src)
        if dst.rank == 0 and dst.world == 1 and not args.no_cpu:
            r["cpu_baseline"] = cpu_baseline(wl, args)
        results[name] = r
        if dst.rank == 0:
            print(f"[bench] {name}: {json.dumps({k: r.get(k) for k in ('value', 'phases', 'e2e')})}", file=sys.stderr,
                  flush=True)
        wl.release()
        del wl
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    head = results[names[0]]
    if dst.rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": "Gint/s", "n_gpus": dst.world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": head["scaling"], "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded splitmix64 generators standing in for BASELINE.json configs)",
            "config": head["config"], "phases": head["phases"], "roofline": head["roofline"],
            "e2e": head.get("e2e"), "gpu_launches": head["gpu_launches"], "clocks": head["clocks"],
            "cpu_baseline": head.get("cpu_baseline"),
        }
        if "gather" in head:
            line["gather"] = head["gather"]
        if len(names) > 1:
            line["workloads"] = {k: v for k, v in results.items() if k != names[0]}
        line["native_libs"] = _loaded_libs()
        print(json.dumps(line), flush=True)
    dev.close()
    dst.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=list(WORKLOADS) + ["all"],
                    help="default: cfg3 headline + the other configs (N=1); cfg5 + cfg4 (N>1)")
    ap.add_argument("--no-extra", action="store_true", help="only the headline workload")
    ap.add_argument("--n", type=int, default=None, help="override array size (single-array workloads)")
    ap.add_argument("--scale", type=float, default=1.0, help="scale batch workloads (cfg4/cfg5)")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=5.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-paper-mode", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gather", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
