"""Does the GPU have room for two config-3 steps at once?  (dev tool, GPU)

Two CUDA-graph plans over two independent input batches; times R replays of
plan A alone, then A and B alternately on ONE stream (sequential), then A on
stream 1 and B on stream 2 (concurrent).  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    torch.cuda.set_device(0)
    S = bench.build_setup("config3", 0, 1, 0)
    hs, K, B, tab, wl, ctx = S["hs"], S["K"], S["B"], S["tab"], S["wl"], S["ctx"]
    cts2 = [hs.Ciphertext.from_words(ctx, c.words()) for c in S["cts"]]
    mk = lambda cts: hs.Plan(K, cts, S["n"], S["m"], S["k"], wl["variant"], tab["exp"], tab["inv"], bts=B)
    pa, pb = mk(S["cts"]), mk(cts2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 4

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    def seq():
        for _ in range(R):
            pa.run()
            pb.run()

    def conc():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        for _ in range(R):
            pa.run(s1.cuda_stream)
            pb.run(s2.cuda_stream)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_seq = timed(seq)
    t_conc = timed(conc)
    out = dict(replays_per_plan=R, seq_ms_per_step=round(t_seq / (2 * R), 2),
               concurrent_ms_per_step=round(t_conc / (2 * R), 2), speedup=round(t_seq / t_conc, 3))
    # the concurrent words equal the sequential ones
    wa = [c.words() for c in pa.outputs[:2]]
    seq()
    torch.cuda.synchronize()
    out["words_equal"] = all((a == c.words()).all() for a, c in zip(wa, pa.outputs[:2]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
