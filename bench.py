#!/usr/bin/env python
"""Headline benchmark: batched Paillier-2048 encrypt + decrypt of 1M fixed-point values per GPU
(BASELINE.json configs[1]), plus the encrypted matvec of configs[2] as an extra.

    python bench.py --gpus N --steps K --warmup W            (N > 1: one rank per GPU over NCCL -- under the driver's
                                                              torchrun, or re-executed under torch.distributed.run
                                                              by this script when WORLD_SIZE is not set)
    python bench.py --impl reference ...                     (the reference's CPU algorithm on the host cores)
    python bench.py --flr-rows 1000000 --no-matvec --no-ops  (BASELINE configs[3] at full size: the documented
                                                              full-size FLR command; record under profiles/)

A step = one pass of the hot path over one batch: encrypt `count` residues, then decrypt the resulting
ciphertexts (2 * count Paillier operations).  `value` is timed with the inputs already resident in HBM;
`e2e` goes through the C ABI's host-buffer entry points (pinned staging, H2D and D2H inside the timed
region); `e2e_operator_api` is the same workload through the frozen Python operator API, host floats to host
floats, with the obfuscator draws, the codec and the HAFB wire hop inside the timed region.  Every rank
processes its own `count` elements (independent shards, no data-path collective): weak scaling.  `extras`
carries the per-operator rates, the config-3 matvec and one heterogeneous-FLR iteration next to the SAME
iteration timed on the host CPU (oracle/flr_cpu.py, row subsample, decrypted values compared).  Prints ONE JSON
line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
for _p in (ROOT, os.path.join(ROOT, "oracle")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

KEY_BITS = 2048
KEY_SEED = 7
# canonical limb products per operation at key 2048: modmul(L) = 2 L^2 + L with
# 32-bit limbs, modexp(b) = 1.25 b modmuls
LP_ENCRYPT = (1.25 * 2048 + 3) * (2 * 128 * 128 + 128) + 64 * 64
LP_DECRYPT = 2 * (1.25 * 1024 + 3) * (2 * 64 * 64 + 64)
LP_MODMUL = 2 * 128 * 128 + 128


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--count", type=int, default=1_000_000, help="elements per GPU per step")
    ap.add_argument("--cpu-sample", type=int, default=4096, help="elements of the bounded CPU sample")
    ap.add_argument("--no-matvec", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flr", action="store_true")
    ap.add_argument("--no-ops", action="store_true", help="skip the per-operator rates in extras")
    ap.add_argument("--e2e-max-steps", type=int, default=10,
                    help="the host-buffer end-to-end leg times min(--steps, this) steps of 2M operations each")
    ap.add_argument("--no-api", action="store_true", help="skip the operator-API end-to-end leg")
    ap.add_argument("--api-steps", type=int, default=5, help="timed steps of the operator-API end-to-end leg")
    ap.add_argument("--flr-rows", type=int, default=50_000,
                    help="rows of the heterogeneous-FLR extra (BASELINE configs[3] shape, 200 features)")
    ap.add_argument("--flr-iters", type=int, default=2, help="FLR iterations (the last one is reported)")
    ap.add_argument("--flr-devices", default="",
                    help="CUDA device indices of the FLR extra's multi-device backend (default: one per rank of "
                         "--gpus; an index may repeat, e.g. 0,0 exercises the sharded path on one GPU)")
    ap.add_argument("--flr-cpu-rows", type=int, default=512,
                    help="rows of the same FLR iteration timed on the host CPU (0 = skip)")
    ap.add_argument("--check", type=int, default=4096, help="strided elements compared with the CPU oracle")
    return ap.parse_args()


def respawn_under_torchrun(args) -> int:
    """`python bench.py --gpus N` without a launcher: run this script as N ranks, one per GPU, over NCCL."""
    import socket
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def bench_key(product: bool = True):
    """keygen(2048, default_rng(7)) -- the config-2 key -- as the checker's key object (p, q,
    CRT constants).  The GPU arm takes it from the product's own key generation (host Python); the reference arm
    from the oracle's, so that nothing of the product package is on its path.  Same seed, same key."""
    import hebatch_oracle as ho
    if not product:
        return ho.keygen(KEY_BITS, random.Random(KEY_SEED))
    from paper_2107_13797_b200 import paillier
    kp = paillier.keygen(KEY_BITS, paillier.default_rng(KEY_SEED))
    return ho.Key(kp.public.n, kp.private.p, kp.private.q)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "250"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except OSError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0])); smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        busy = [v for v in sm if v > 0.5 * max(smax or [1])] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(smax) if smax else None, "samples": len(sm), "reasons": sorted(reasons)}


def cpu_reference_rate(key, sample: int, rng_seed: int = 1):
    """The reference's CPU algorithm (GMP powm, all host threads) on a bounded sample of the workload."""
    import numpy as np
    import cpuref
    wn, wc = cpuref.widths(key.n)
    rs = np.random.default_rng(rng_seed)
    m = rs.integers(0, 2 ** 32, size=(sample, wn), dtype=np.uint32); m[:, -1] = 0
    r = rs.integers(0, 2 ** 32, size=(sample, wn), dtype=np.uint32); r[:, -1] = 1
    threads = cpuref.threads()
    t0 = time.perf_counter()
    c = cpuref.encrypt_words(key.n, m, r, threads)
    t1 = time.perf_counter()
    back = cpuref.decrypt_words(key, c, threads)
    t2 = time.perf_counter()
    if not (back == m).all():
        raise RuntimeError("CPU reference round trip failed")
    return {"ops_per_s": 2 * sample / (t2 - t0), "encrypt_per_s": sample / (t1 - t0),
            "decrypt_per_s": sample / (t2 - t1), "seconds": t2 - t0, "threads": threads}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    key = bench_key(product=False)
    sample = args.cpu_sample
    for _ in range(args.warmup):
        cpu_reference_rate(key, max(64, sample // 16))
    times, last = [], None
    for _ in range(args.steps):
        last = cpu_reference_rate(key, sample)
        times.append(last["seconds"])
    total = sum(times)
    value = 2 * sample * args.steps / total
    line = {
        "impl": "reference", "metric": "paillier2048_encrypt_decrypt_ops_per_s", "value": value,
        "unit": "ops/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "batched Paillier-2048 encrypt + decrypt (BASELINE configs[1])",
                   "key_bits": KEY_BITS, "count_per_step": sample,
                   "note": "bounded sample of the 1M-element workload; per-element cost is uniform"},
        "cpu_baseline": {"value": value, "unit": "ops/s", "cores": last["threads"], "kind": "port",
                         "sample": f"{sample} encrypt + {sample} decrypt per step, GMP mpz_powm under OpenMP "
                                   "(oracle/cpu_ref.c), the arithmetic the reference reaches through gmpy2"},
        "e2e": {"value": value, "unit": "ops/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def measured_imad_peak():
    """Live integer-multiply peak (LP/s) from the standalone microbenchmark; falls back to the committed one."""
    exe = os.path.join(ROOT, "build", "imad_peak2")
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120, check=True).stdout
        data = json.loads(out.strip().splitlines()[-1])
        return data["lp_per_s_wide_carry"], "measured live (build/imad_peak2, IMAD.WIDE.U32.X chains)"
    except Exception:
        with open(os.path.join(ROOT, "profiles", "r01_imad_peak2.json")) as fh:
            data = json.load(fh)
        return data["lp_per_s_wide_carry"], "profiles/r01_imad_peak2.json (earlier run on this pool)"


def strided_check(key, m, r, c, back, count, nchk):
    """Ciphertexts and decryptions of `nchk` elements spread over the whole batch against the CPU oracle (GMP),
    bit for bit -- the reference verifies min(count, 4096) elements itself (cli.py:204).  The same CPU pass is the
    cpu_baseline sample: it returns the oracle's rates."""
    import numpy as np
    import torch
    import cpuref
    nchk = max(1, min(nchk, count))
    idx = torch.arange(nchk, device=m.device, dtype=torch.int64) * (count // nchk)
    hm = m[idx].cpu().numpy().view(np.uint32)
    hr = r[idx].cpu().numpy().view(np.uint32)
    hc = c[idx].cpu().numpy().view(np.uint32)
    threads = cpuref.threads()
    t0 = time.perf_counter()
    want = cpuref.encrypt_words(key.n, hm, hr, threads)
    t1 = time.perf_counter()
    dec = cpuref.decrypt_words(key, want, threads)
    t2 = time.perf_counter()
    if not np.array_equal(want, hc):
        raise SystemExit("ciphertexts differ from the CPU oracle")
    if not np.array_equal(dec, hm) or not np.array_equal(back[idx].cpu().numpy().view(np.uint32), hm):
        raise SystemExit("decryptions differ from the CPU oracle")
    return {"ops_per_s": 2 * nchk / (t2 - t0), "encrypt_per_s": nchk / (t1 - t0), "decrypt_per_s": nchk / (t2 - t1),
            "seconds": t2 - t0, "threads": threads, "sample": nchk}


def operator_api_e2e(key, count, steps, rank):
    """The workload through the frozen operator API (operators.py:109-167 of the reference), host floats in, host
    floats out: batch_encode -> batch_encrypt(pk, plain, random.Random(seed)) -> serialize_to_bytes -> deserialize
    -> batch_decrypt -> batch_decode.  Obfuscator draws (MT19937 replay + gcd test), codec, batch objects and
    the HAFB hop are inside the timed region."""
    import numpy as np
    import torch
    from paper_2107_13797_b200 import operators as ops, paillier
    from paper_2107_13797_b200.bufferpool import deserialize, serialize_to_bytes
    kp = paillier.keypair_from_primes(key.p, key.q)
    pk, sk = kp.public, kp.private
    vals = np.random.default_rng(77 + rank).uniform(-100.0, 100.0, count)
    grid = np.round(vals * 4294967296.0) / 4294967296.0            # exponent -8: the 16^-8 = 2^-32 grid

    def api_step(seed):
        plain = ops.batch_encode(pk, vals, -8)
        cipher = ops.batch_encrypt(pk, plain, random.Random(seed))
        wire = serialize_to_bytes(cipher)
        back = ops.batch_decrypt(sk, deserialize(wire, pk))
        return ops.batch_decode(pk, back), len(wire)

    out, wire_len = api_step(1)
    if not np.array_equal(np.asarray(out), grid):
        raise SystemExit("operator API round trip is not the grid-rounded input")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        out, _ = api_step(2 + i)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if not np.array_equal(np.asarray(out), grid):
        raise SystemExit("operator API round trip is not the grid-rounded input")
    return dt, wire_len


def run_b200(args):
    import numpy as np
    import torch
    from paper_2107_13797_b200 import _native, device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # Rehearsal of the multi-rank code path on a box with fewer GPUs than ranks (development only; the numbers mean
    # nothing): HB_BENCH_SHARE_DEVICES=1 maps rank r to device r mod device_count and the collectives go over gloo
    # on host tensors, because NCCL refuses two ranks on one device.
    rehearsal = os.environ.get("HB_BENCH_SHARE_DEVICES", "") not in ("", "0")
    ndev = torch.cuda.device_count()
    if local >= ndev and not rehearsal:
        raise SystemExit(f"rank {rank} needs CUDA device {local}, the box has {ndev}")
    local = local % ndev
    torch.cuda.set_device(local)
    dist = None
    comm_dev = "cpu" if rehearsal else "cuda"
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        if rehearsal:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=comm_dev)
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    key = bench_key()
    lib = _native.lib()
    ctx = device.context_for(key.n)
    ctx.set_private(key.p, key.q, key.hp, key.hq, key.q_inv)
    wn, wc = ctx.wn, ctx.wc
    count = args.count
    stream = device.current_stream_ptr()

    # synthetic residues: config 2 encodes uniform(-100, 100) at exponent -8 (39-bit magnitudes, half of them
    # negative residues n - |x|): produced by the device codec, seeded per rank
    g = torch.Generator(device="cuda"); g.manual_seed(1234 + rank)
    vals = (torch.rand(count, generator=g, device="cuda", dtype=torch.float64) * 200.0 - 100.0)
    m = torch.empty((count, wn), dtype=torch.int32, device="cuda")
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    _native.check(lib.hb_encode_f64(ctx.handle, vals.data_ptr(), -8, m.data_ptr(), count, bad.data_ptr(), stream))
    # obfuscation factors: uniform below 2^(key_bits - 32) < n (gcd with n is 1 with overwhelming probability).
    # The reference's own draw (draw_unit) is timed inside `e2e_operator_api`, not here.
    r = torch.randint(-2 ** 31, 2 ** 31 - 1, (count, wn), generator=g, device="cuda", dtype=torch.int32)
    r[:, -1] = 1
    c = torch.empty((count, wc), dtype=torch.int32, device="cuda")
    back = torch.empty((count, wn), dtype=torch.int32, device="cuda")

    def step():
        _native.check(lib.hb_encrypt(ctx.handle, m.data_ptr(), r.data_ptr(), c.data_ptr(), count, stream))
        _native.check(lib.hb_decrypt(ctx.handle, c.data_ptr(), back.data_ptr(), count, stream))

    for _ in range(args.warmup):
        step()
    barrier()
    if not torch.equal(back, m):
        raise SystemExit("round trip failed: decrypt(encrypt(m)) != m")
    # parity at the benchmarked shape: `--check` strided elements against the CPU oracle (GMP), on rank 0; the same
    # pass is the bounded CPU sample of cpu_baseline
    cpu = strided_check(key, m, r, c, back, count, args.check) if rank == 0 else None

    sampler = ClockSampler(local)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    launches0 = device.launch_count()
    barrier()
    sampler.start()
    enc_ms = dec_ms = 0.0
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_start.record()
    for _ in range(args.steps):
        ev[0].record()
        _native.check(lib.hb_encrypt(ctx.handle, m.data_ptr(), r.data_ptr(), c.data_ptr(), count, stream))
        ev[1].record()
        _native.check(lib.hb_decrypt(ctx.handle, c.data_ptr(), back.data_ptr(), count, stream))
        ev[2].record()
        ev[2].synchronize()
        enc_ms += ev[0].elapsed_time(ev[1])
        dec_ms += ev[1].elapsed_time(ev[2])
    e_end.record()
    barrier()
    clocks = sampler.stop()
    launches = device.launch_count() - launches0
    elapsed_ms = max_over_ranks(e_start.elapsed_time(e_end))
    ms_per_step = elapsed_ms / args.steps
    value = 2.0 * count * world / (ms_per_step * 1e-3)

    # ---- end to end through the host-buffer C ABI (rank-local shard, pinned staging inside the library)
    e2e = None
    if not args.no_e2e:
        hm = m.cpu().numpy().view(np.uint32)
        hr = r.cpu().numpy().view(np.uint32)
        hc = np.empty((count, wc), np.uint32)
        hb = np.empty((count, wn), np.uint32)

        def host_step():
            _native.check(lib.hb_encrypt_host(ctx.handle, hm.ctypes.data, hr.ctypes.data, hc.ctypes.data, count))
            _native.check(lib.hb_decrypt_host(ctx.handle, hc.ctypes.data, hb.ctypes.data, count))

        host_step()
        barrier()
        e2e_steps = max(1, min(args.steps, args.e2e_max_steps))      # bounded so that a --steps 20 run stays within minutes
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            host_step()
        barrier()
        dt = max_over_ranks(time.perf_counter() - t0)
        if not np.array_equal(hb, hm):
            raise SystemExit("host-path round trip failed")
        e2e = {"value": 2.0 * count * world * e2e_steps / dt, "unit": "ops/s",
               "h2d_bytes_per_step": int(count * (2 * wn + wc) * 4), "d2h_bytes_per_step": int(count * (wc + wn) * 4),
               "steps": e2e_steps, "api": "hb_encrypt_host + hb_decrypt_host (include/hebatch_b200.h)"}
        del hm, hr, hc, hb

    # ---- the same workload through the frozen operator API, host floats to host floats
    api = None
    if not args.no_api:
        api_steps = max(1, args.api_steps)
        barrier()
        dt, wire_len = operator_api_e2e(key, count, api_steps, rank)
        dt = max_over_ranks(dt)
        api = {"value": 2.0 * count * world * api_steps / dt, "unit": "ops/s", "steps": api_steps,
               "ms_per_step": 1e3 * dt / api_steps,
               "h2d_bytes_per_step": int(count * (8 + 4 * wn) + wire_len), "d2h_bytes_per_step": int(wire_len + 8 * count),
               "api": "batch_encode -> batch_encrypt(random.Random(seed)) -> serialize_to_bytes -> deserialize -> "
                      "batch_decrypt -> batch_decode; draws, codec and the HAFB hop inside the timed region"}

    extras = {"encrypt_per_s_per_gpu": count * args.steps / (enc_ms * 1e-3),
              "decrypt_per_s_per_gpu": count * args.steps / (dec_ms * 1e-3)}

    # ---- extra: encrypted matvec, BASELINE configs[2] (100k x 100, sharded by rows across ranks)
    if not args.no_matvec and count >= 100_000:
        inner, d = 100_000 // world, 100
        xg = torch.rand(inner * d, generator=g, device="cuda", dtype=torch.float64) * 2.0 - 1.0
        xk = torch.empty((inner * d, wn), dtype=torch.int32, device="cuda")
        _native.check(lib.hb_encode_f64(ctx.handle, xg.data_ptr(), -13, xk.data_ptr(), inner * d, bad.data_ptr(), stream))
        mv = torch.empty((d, wc), dtype=torch.int32, device="cuda")
        ab = torch.empty((2 * d, wc), dtype=torch.int32, device="cuda")

        def matvec_once():
            if world == 1:
                _native.check(lib.hb_matvec(ctx.handle, c.data_ptr(), xk.data_ptr(), mv.data_ptr(), 1, inner, d, stream))
                return
            # rows are sharded: per-rank partial pairs, NCCL all-gather (d x 2 ciphertexts per rank), combine
            _native.check(lib.hb_matvec_partial(ctx.handle, c.data_ptr(), xk.data_ptr(), ab.data_ptr(), inner, d, stream))
            mine = ab.to(comm_dev)
            parts = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(parts, mine)
            allab = torch.cat(parts, dim=0).to("cuda").contiguous()
            _native.check(lib.hb_matvec_combine(ctx.handle, allab.data_ptr(), world, mv.data_ptr(), d, stream))

        matvec_once()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        reps = 3
        for _ in range(reps):
            matvec_once()
        b.record()
        barrier()
        mv_ms = max_over_ranks(a.elapsed_time(b) / reps)
        terms = 100_000 // world * world * d
        extras["matvec_100k_x_100_ms"] = mv_ms
        extras["matvec_terms_per_s"] = terms / (mv_ms * 1e-3)
        # canonical work: (1.25 * 52 + 1) modmuls per term (SURVEY.md 8d, 52-bit scalars)
        extras["matvec_canonical_lp_per_s"] = terms * (1.25 * 52 + 1) * LP_MODMUL / (mv_ms * 1e-3)
        if rank == 0:
            # ciphertext-for-ciphertext against the CPU oracle on the reduced instance SURVEY 8d names: 2000 x 100
            import cpuref
            sub = 2000
            mv2 = torch.empty((d, wc), dtype=torch.int32, device="cuda")
            _native.check(lib.hb_matvec(ctx.handle, c.data_ptr(), xk.data_ptr(), mv2.data_ptr(), 1, sub, d, stream))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            want = cpuref.matvec_words(key.n, c[:sub].cpu().numpy().view(np.uint32),
                                       xk[:sub * d].cpu().numpy().view(np.uint32), sub, d)
            cpu_mv_s = time.perf_counter() - t0
            if not np.array_equal(want, mv2.cpu().numpy().view(np.uint32)):
                raise SystemExit("matvec differs from the CPU oracle")
            extras["matvec_oracle_check"] = f"{sub} x {d}: bit-identical"
            extras["matvec_cpu_terms_per_s"] = sub * d / cpu_mv_s
        del xg, xk

    # ---- extra: the other six operators of the reference's own harness (bench.py:65-101 of the reference:
    # encode, decode, hmul, hadd, hsum next to henc / hdec / hmatmul), each on this rank's `count` elements.
    # Ciphertext operators are timed in BOTH forms the library keeps ciphertexts in: plain words (the wire form;
    # what a single stand-alone call sees) and Montgomery digits (the resident form chained operators see).
    if not args.no_ops:
        def timed(fn, reps=2):
            fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            b.synchronize()
            return a.elapsed_time(b) * 1e-3 / reps

        A, B, O = 0x10, 0x20, 0x40
        lc = int(lib.hb_ct_limbs(ctx.handle))
        tmp_c = torch.empty((count, max(wc, lc)), dtype=torch.int32, device="cuda")
        tmp_m = torch.empty((count, wn), dtype=torch.int32, device="cuda")
        tmp_f = torch.empty(count, dtype=torch.float64, device="cuda")
        one_c = torch.empty((1, max(wc, lc)), dtype=torch.int32, device="cuda")
        cm = torch.empty((count, lc), dtype=torch.int32, device="cuda")
        _native.check(lib.hb_ct_convert(ctx.handle, c.data_ptr(), cm.data_ptr(), count, 1, stream))
        t_enc = timed(lambda: _native.check(lib.hb_encode_f64(ctx.handle, vals.data_ptr(), -8, tmp_m.data_ptr(), count,
                                                              bad.data_ptr(), stream)), reps=20)
        t_dec = timed(lambda: _native.check(lib.hb_decode_f64(ctx.handle, m.data_ptr(), -8, tmp_f.data_ptr(), count,
                                                              bad.data_ptr(), stream)), reps=20)
        if not torch.equal(tmp_m, m):
            raise SystemExit("codec is not deterministic")
        grid = torch.round(vals * 4294967296.0) / 4294967296.0          # exponent -8: the 16^-8 = 2^-32 grid
        if not torch.equal(tmp_f, grid):
            raise SystemExit("decode(encode(v)) is not v rounded to the 16^-8 grid")
        t_add = timed(lambda: _native.check(lib.hb_mulmod(ctx.handle, c.data_ptr(), c.data_ptr(), tmp_c.data_ptr(),
                                                          count, 0, stream)))
        t_add_m = timed(lambda: _native.check(lib.hb_mulmod_rep(ctx.handle, cm.data_ptr(), cm.data_ptr(),
                                                                tmp_c.data_ptr(), count, 0, A | B | O, stream)))
        # scalars = the encoded values themselves: 39-bit magnitudes, half of them negative residues (inverse base)
        t_mul = timed(lambda: _native.check(lib.hb_powscalar(ctx.handle, c.data_ptr(), m.data_ptr(), tmp_c.data_ptr(),
                                                             count, count, 0, stream)), reps=1)
        t_mul_m = timed(lambda: _native.check(lib.hb_powscalar(ctx.handle, cm.data_ptr(), m.data_ptr(), tmp_c.data_ptr(),
                                                               count, count, A | O, stream)), reps=1)
        t_sum = timed(lambda: _native.check(lib.hb_product(ctx.handle, c.data_ptr(), one_c.data_ptr(), 1, count, 0, 1,
                                                           stream)))
        t_sum_m = timed(lambda: _native.check(lib.hb_product_rep(ctx.handle, cm.data_ptr(), one_c.data_ptr(), 1, count,
                                                                 0, 1, A | O, stream)))
        codec_bytes = count * (8 + 4 * wn)
        extras["operators_per_s_per_gpu"] = {
            "encode": count / t_enc, "decode": count / t_dec, "hadd": count / t_add, "hmul_39bit_signed": count / t_mul,
            "hsum_elements": count / t_sum, "hadd_resident": count / t_add_m,
            "hmul_39bit_signed_resident": count / t_mul_m, "hsum_elements_resident": count / t_sum_m}
        extras["codec_hbm_frac"] = {"encode": codec_bytes / t_enc / 1e9 / _hbm_peak(),
                                    "decode": codec_bytes / t_dec / 1e9 / _hbm_peak()}
        del tmp_c, tmp_m, tmp_f, cm
        # the codec again at 8M elements (2 GiB of residues): well beyond the 126 MB L2, where the 1M-element figure
        # above is flattered by write-back and hurt by the launch tail of a 50 us kernel
        big = 8 * count
        if big * 4 * wn <= 4 << 30:
            vbig = torch.rand(big, generator=g, device="cuda", dtype=torch.float64) * 200.0 - 100.0
            mbig = torch.empty((big, wn), dtype=torch.int32, device="cuda")
            fbig = torch.empty(big, dtype=torch.float64, device="cuda")
            tb_enc = timed(lambda: _native.check(lib.hb_encode_f64(ctx.handle, vbig.data_ptr(), -8, mbig.data_ptr(), big,
                                                                   bad.data_ptr(), stream)), reps=10)
            tb_dec = timed(lambda: _native.check(lib.hb_decode_f64(ctx.handle, mbig.data_ptr(), -8, fbig.data_ptr(), big,
                                                                   bad.data_ptr(), stream)), reps=10)
            if not torch.equal(fbig, torch.round(vbig * 4294967296.0) / 4294967296.0):
                raise SystemExit("decode(encode(v)) is not v rounded to the 16^-8 grid (8M elements)")
            big_bytes = big * (8 + 4 * wn)
            extras["codec_beyond_l2"] = {"elements": big, "encode_per_s": big / tb_enc, "decode_per_s": big / tb_dec,
                                         "encode_gbs": big_bytes / tb_enc / 1e9, "decode_gbs": big_bytes / tb_dec / 1e9,
                                         "encode_hbm_frac": big_bytes / tb_enc / 1e9 / _hbm_peak(),
                                         "decode_hbm_frac": big_bytes / tb_dec / 1e9 / _hbm_peak()}
            del vbig, mbig, fbig

    del m, r, c, back, vals
    torch.cuda.empty_cache()
    barrier()
    if dist is not None:
        dist.destroy_process_group()
    if rank != 0:
        return

    # ---- extra (rank 0): one full-batch iteration of heterogeneous FLR (BASELINE configs[3] shape at --flr-rows),
    # on all `world` GPUs through the single-process multi-device backend (the parties are sequential state
    # machines: the GPUs of the box serve one party's operator call at a time), next to the same
    # iteration on the host CPU
    if not args.no_flr and count >= 100_000:
        if world > 1:
            time.sleep(2.0)                      # the other ranks are leaving their GPUs
        devices = ([int(v) for v in args.flr_devices.split(",")] if args.flr_devices
                   else [d % ndev for d in range(world)])
        extras.update(flr_extra(args.flr_rows, devices, args.flr_iters))
        if args.flr_cpu_rows > 0:
            extras.update(flr_cpu_extra(args.flr_cpu_rows, extras["flr_hetero_iter_s"], args.flr_rows))

    peak, peak_src = measured_imad_peak()
    enc_s = enc_ms * 1e-3 / args.steps            # average k_encrypt launch duration (one launch per step)
    achieved = LP_ENCRYPT * count / enc_s
    roofline = {
        "bound": "imad", "kernel": "k_encrypt<32,4>", "achieved": achieved / 1e12, "peak": peak / 1e12,
        "unit": "TLP/s (1e12 32x32->64 limb products per second)", "frac": achieved / peak,
        "traffic": _ncu_traffic_per_element() * count if _ncu_traffic_per_element() else None,
        "peak_source": peak_src,
        "note": "integer-multiply bound, not HBM: algorithmic bytes per encrypt are 1 KiB against 8.4e7 limb products",
        "hbm": {"achieved_gbs": count * (2 * wn + wc) * 4 / enc_s / 1e9, "peak_gbs": _hbm_peak()},
        "decrypt_frac": (LP_DECRYPT * count / (dec_ms * 1e-3 / args.steps)) / peak,
    }
    if "matvec_canonical_lp_per_s" in extras:
        roofline["matvec_frac_canonical"] = extras["matvec_canonical_lp_per_s"] / peak
    if "operators_per_s_per_gpu" in extras:
        rates = extras["operators_per_s_per_gpu"]
        lp_hmul = (1.25 * 39 + 1) * LP_MODMUL
        roofline["operator_frac_canonical"] = {
            "hadd": rates["hadd"] * LP_MODMUL / peak, "hadd_resident": rates["hadd_resident"] * LP_MODMUL / peak,
            "hmul": rates["hmul_39bit_signed"] * lp_hmul / peak,
            "hmul_resident": rates["hmul_39bit_signed_resident"] * lp_hmul / peak,
            "hsum": rates["hsum_elements"] * LP_MODMUL / peak,
            "hsum_resident": rates["hsum_elements_resident"] * LP_MODMUL / peak}
    line = {
        "metric": "paillier2048_encrypt_decrypt_ops_per_s", "value": value, "unit": "ops/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "batched Paillier-2048 encrypt + decrypt of 1M fixed-point values per GPU "
                               "(BASELINE configs[1])",
                   "key_bits": KEY_BITS, "count_per_gpu": count, "parallelism": f"shard{world}",
                   "l2": "inputs per step (1 GiB) exceed the 126 MB L2; no explicit flush",
                   "oracle_check": f"{cpu['sample']} strided elements: ciphertexts and decryptions bit-identical "
                                   "to the CPU oracle"},
        **({"rehearsal": "ranks share devices, gloo collectives: code-path check only, not a measurement"}
           if rehearsal else {}),
        "clocks": clocks, "e2e": e2e, "e2e_operator_api": api, "gpu_launches": launches, "roofline": roofline,
        "cpu_baseline": {"value": cpu["ops_per_s"], "unit": "ops/s", "cores": cpu["threads"], "kind": "port",
                         "sample": f"{cpu['sample']} encrypt + {cpu['sample']} decrypt of the benchmarked batch, GMP "
                                   f"mpz_powm under OpenMP (oracle/cpu_ref.c); encrypt {cpu['encrypt_per_s']:.1f}/s, "
                                   f"decrypt {cpu['decrypt_per_s']:.1f}/s"},
        "extras": extras,
    }
    print(json.dumps(line), flush=True)


def flr_extra(rows: int, devices=(0,), iters: int = 2, features: int = 200):
    """Full-batch iterations (gradient step + loss over all rows) of 2-party heterogeneous FLR through the
    package's operator API at Paillier-2048; the last one is reported (the first also encodes the feature
    matrices, which stay resident).  Per iteration: 5 * rows full-width modular powers, two rows x ~100 encrypted
    matvecs, ~3 * rows scalar powers, ~4 * rows modular products, 202 decryptions.  With more than one device the
    operators run on the single-process multi-device backend (element shards per device, matvec partials
    combined on the first device)."""
    import numpy as np
    import torch
    from paper_2107_13797_b200 import flr, paillier
    from paper_2107_13797_b200.backends import MultiDeviceBackend
    ids, X, y = flr.make_synthetic(rows, features, seed=42)
    guest, host = flr.vertical_split(ids, X, y, 2)
    keys = paillier.keygen(KEY_BITS, paillier.default_rng(KEY_SEED), allow_insecure=True)
    devices = list(devices)
    backend = MultiDeviceBackend(devices) if len(devices) > 1 else None
    fed = flr.HeteroFederation(guest, host, [np.arange(rows)], np.arange(rows), keys,
                               flr.FlrConfig(0.15, rows, seed=42), backend=backend)
    secs, losses = [], []
    for _ in range(max(2, iters)):
        for dev in set(devices):
            torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        res = fed.run_epoch()
        for dev in set(devices):
            torch.cuda.synchronize(dev)
        secs.append(time.perf_counter() - t0)
        losses.append(res.loss)
    if not (losses[1] < losses[0] < 0.6932):
        raise SystemExit(f"FLR loss did not decrease: {losses}")
    if backend is not None:
        backend.close()
    return {"flr_hetero_iter_s": secs[-1], "flr_first_iter_s": secs[0], "flr_iter_s_all": secs, "flr_rows": rows,
            "flr_features": features, "flr_devices": len(devices), "flr_device_ids": devices,
            "flr_modexp_per_iter": 5 * rows + 2 * (features + 1) + 1, "flr_loss": losses}


def flr_cpu_extra(cpu_rows: int, gpu_iter_s: float, gpu_rows: int, features: int = 200):
    """The same FLR iteration on the host CPU (oracle/flr_cpu.py: the reference's protocol with every modular
    power in GMP under OpenMP on all host threads), MEASURED on a row subsample and scaled linearly in rows (every
    per-iteration operator count is linear in rows except the 202 decryptions).  The GPU path runs the same
    subsample with the same data, key and seeds, and everything the arbiter decrypts -- masked gradients, loss --
    must be equal."""
    import numpy as np
    import flr_cpu
    import hebatch_oracle as ho
    from paper_2107_13797_b200 import flr, paillier
    ids, X, y = flr.make_synthetic(cpu_rows, features, seed=42)
    guest, host = flr.vertical_split(ids, X, y, 2)
    keys = paillier.keygen(KEY_BITS, paillier.default_rng(KEY_SEED), allow_insecure=True)
    fed = flr.HeteroFederation(guest, host, [np.arange(cpu_rows)], np.arange(cpu_rows), keys,
                               flr.FlrConfig(0.15, cpu_rows, seed=42))
    okey = ho.Key(keys.public.n, keys.private.p, keys.private.q)
    ref = flr_cpu.CpuHeteroFlr(okey, guest.X, guest.y, host.X, 0.15, 42)
    gpu_losses, cpu_losses, cpu_secs = [], [], []
    for _ in range(2):
        gpu_losses.append(fed.run_epoch().loss)
        cpu_losses.append(ref.run_iteration())
        cpu_secs.append(dict(ref.seconds))
    if gpu_losses != cpu_losses or fed.decrypted != ref.decrypted:
        raise SystemExit("FLR iteration differs from the host-CPU reference iteration")
    last = cpu_secs[-1]
    scaled = last["total"] * gpu_rows / cpu_rows
    return {"flr_cpu_iter_s": scaled, "flr_cpu_sample_rows": cpu_rows, "flr_cpu_sample_iter_s": last["total"],
            "flr_cpu_cores": ref.threads, "flr_cpu_breakdown_s": {k: round(v, 4) for k, v in last.items()},
            "flr_speedup_vs_cpu": scaled / gpu_iter_s,
            "flr_cpu_check": f"{cpu_rows}-row iteration x2: every decrypted gradient and the loss equal on GPU and CPU",
            "flr_cpu_note": "CPU time measured on the row subsample, scaled linearly to flr_rows"}


def _ncu_traffic_per_element():
    """dram bytes read + written per encrypted element, from the committed ncu --set full capture of k_encrypt
    (profiles/r02_ncu_summary.json; the capture ran 37888 elements).  Almost all of it is the per-warp window
    tables (33 slots x 4 KiB per warp, 160 MB for the grid: more than the L2 holds), not operand traffic -- about
    8 GB/s, a thousandth of the HBM bandwidth, under a multiplier-bound kernel."""
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_summary.json")) as fh:
            enc = json.load(fh)["encrypt"]
        total = sum(float(enc[k]["value"]) * scale[enc[k]["unit"]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        return total / 37888
    except Exception:
        return None


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)["hbm_gbs"]
    except Exception:
        return 6650.0


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(respawn_under_torchrun(args))
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
