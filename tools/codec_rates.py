"""Codec rates (hb_encode_f64 / hb_decode_f64) against the HBM roofline, at a size beyond the L2 (development and
profiling tool, GPU box).  264 algorithmic bytes per element at 2048-bit keys (8 B of double + one residue).

    python tools/codec_rates.py --key-bits 2048 --count 8000000 [--lib alt.so]
"""
import argparse
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--key-bits", type=int, default=2048)
    ap.add_argument("--count", type=int, default=8_000_000)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--lib", default="")
    args = ap.parse_args()
    import torch
    import hebatch_oracle as ho
    from paper_2107_13797_b200 import _native, device
    if args.lib:
        _native.LIB_PATH = os.path.abspath(args.lib)
    key = ho.keygen(args.key_bits, random.Random(7))
    lib = _native.lib()
    ctx = device.context_for(key.n)
    wn = ctx.wn
    count = args.count
    stream = device.current_stream_ptr()
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    vals = torch.rand(count, generator=g, device="cuda", dtype=torch.float64) * 200.0 - 100.0
    m = torch.empty((count, wn), dtype=torch.int32, device="cuda")
    back = torch.empty(count, dtype=torch.float64, device="cuda")
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) * 1e-3 / args.reps

    t_enc = timed(lambda: _native.check(lib.hb_encode_f64(ctx.handle, vals.data_ptr(), -8, m.data_ptr(), count,
                                                          bad.data_ptr(), stream)))
    t_dec = timed(lambda: _native.check(lib.hb_decode_f64(ctx.handle, m.data_ptr(), -8, back.data_ptr(), count,
                                                          bad.data_ptr(), stream)))
    grid = torch.round(vals * 4294967296.0) / 4294967296.0
    ok = bool(torch.equal(back, grid)) and int(bad.item()) == -1
    # the residues themselves, against Python integers, on a strided sample
    idx = list(range(0, count, max(1, count // 64)))[:64]
    rows = m[idx].cpu().numpy().view("uint32")
    for i, row in zip(idx, rows):
        want = ho.encode(key, float(vals[i].item()), -8)[0]
        if int.from_bytes(row.tobytes(), "little") != want:
            ok = False
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        hbm = json.load(fh)["hbm_gbs"]
    nbytes = count * (8 + 4 * wn)
    print(json.dumps({"key_bits": args.key_bits, "count": count, "correct": ok,
                      "encode_per_s": count / t_enc, "decode_per_s": count / t_dec,
                      "encode_gbs": nbytes / t_enc / 1e9, "decode_gbs": nbytes / t_dec / 1e9,
                      "hbm_copy_peak_gbs": hbm, "encode_frac": nbytes / t_enc / 1e9 / hbm,
                      "decode_frac": nbytes / t_dec / 1e9 / hbm}))


if __name__ == "__main__":
    main()
