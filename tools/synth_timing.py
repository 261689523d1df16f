"""Time generate_synthetic on the device (rsim_synth_generate, end to end with the host copies of
the columns) against the host generator and the reference's own (--ref, this container only)
for the config-4 spec (1M requests). Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_15202_b200 import workloads as W  # noqa: E402
from paper_2603_15202_b200.trace import generate_synthetic_device, generate_synthetic_packed  # noqa: E402


def best(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), out


def main():
    spec = W.chat_spec(1_000_000, 12288.0, 0)
    generate_synthetic_device(W.chat_spec(1000, 48.0, 0))          # context + module load
    dev, a = best(lambda: generate_synthetic_device(spec), 5)
    import ctypes as C
    from paper_2603_15202_b200 import _native
    L = _native.lib()
    arr = (_native.SynthClass * len(spec.classes))(*[_native.SynthClass(c.weight, c.shared_blocks, *c.suffix_blocks,
                                                                         *c.output_tokens) for c in spec.classes])

    def gen_only():
        g = C.c_void_p()
        assert L.rsim_synth_generate(C.cast(arr, C.c_void_p), len(spec.classes), spec.duration_s,
                                     spec.mean_rate_rps, spec.seed, spec.block_size, 0, C.byref(g), None, None) == 0
        L.rsim_synth_free(g)
    gen, _ = best(gen_only, 5)
    host, b = best(lambda: generate_synthetic_packed(spec), 1)
    same = all((getattr(a, c).view("u8") == getattr(b, c).view("u8")).all() for c in
               ("request_id", "arrival_s", "in_tokens", "out_tokens", "class_key", "blk_off", "blocks"))
    print(json.dumps({"spec": "config4 chat mix, 1M requests", "n": len(a), "n_blocks": int(a.blk_off[-1]),
                      "device_s": round(dev, 4), "device_generate_only_s": round(gen, 4), "host_numpy_s": round(host, 3), "identical": bool(same)}))


if __name__ == "__main__":
    main()
