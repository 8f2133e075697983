"""Diagnostic: schedules for the per-step host round trip of the cfg2 parameters
(9.6 MB: geometry + opacity 4.8 MB, amplitude/phase 4.8 MB) around a
sleep-kernel stand-in for the 1 ms device step (binning 77 us, then the rest).

  base     : the device step only
  current  : run_host's schedule (geometry D2H at the end of step k; H2D of it
             at the start of k+1 alongside the amplitude/phase D2H, whose H2D
             follows; only the post-binning part waits for amplitude/phase)
  pieces P : the same ranges as P pieces each, every piece's H2D issued as its
             D2H lands (second copy stream), geometry at the end of step k
Each schedule runs eagerly on streams and as one CUDA graph per step.
"""
import time

import torch

MB = 1 << 20
N_GEO = int(4.8e6) // 4  # floats
N_AP = int(4.8e6) // 4
CLK = 1.9e9


def main():
    dev = torch.device("cuda")
    d = torch.zeros(N_GEO + N_AP, device=dev)
    h = torch.zeros(N_GEO + N_AP, pin_memory=True)
    st, c1, c2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    bin_cyc, rest_cyc = int(77e-6 * CLK), int(923e-6 * CLK)

    def rt(src_stream, off, n, pieces, done_stream):
        """D2H of [off, off+n) on c2 in pieces, each piece's H2D on c1 after it."""
        e = torch.cuda.Event()
        e.record(src_stream)
        c2.wait_event(e)
        c1.wait_event(e)
        step = (n + pieces - 1) // pieces
        for o in range(0, n, step):
            m = min(step, n - o)
            with torch.cuda.stream(c2):
                h[off + o:off + o + m].copy_(d[off + o:off + o + m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(c2)
            c1.wait_event(ev)
            with torch.cuda.stream(c1):
                d[off + o:off + o + m].copy_(h[off + o:off + o + m], non_blocking=True)
        fin = torch.cuda.Event()
        fin.record(c1)
        done_stream.wait_event(fin)
        return fin

    def step(kind, first):
        with torch.cuda.stream(st):
            if kind == "base":
                torch.cuda._sleep(bin_cyc)
                torch.cuda._sleep(rest_cyc)
                return
            if kind == "current":
                fork = torch.cuda.Event()
                fork.record(st)
                if not first:
                    c2.wait_event(fork)
                    with torch.cuda.stream(c2):
                        h[N_GEO:].copy_(d[N_GEO:], non_blocking=True)
                    apd = torch.cuda.Event()
                    apd.record(c2)
                h[:N_GEO]  # geometry H2D on st
                d[:N_GEO].copy_(h[:N_GEO], non_blocking=True)
                f2 = torch.cuda.Event()
                f2.record(st)
                c1.wait_event(f2)
                if not first:
                    c1.wait_event(apd)
                with torch.cuda.stream(c1):
                    d[N_GEO:].copy_(h[N_GEO:], non_blocking=True)
                ap = torch.cuda.Event()
                ap.record(c1)
                torch.cuda._sleep(bin_cyc)
                st.wait_event(ap)
                torch.cuda._sleep(rest_cyc)
                h[:N_GEO].copy_(d[:N_GEO], non_blocking=True)
                return
            pieces = int(kind.split()[1])
            if first:
                d.copy_(h, non_blocking=True)
                ap_done = None
            else:
                # amplitude/phase round trip alongside binning
                ap_done = torch.cuda.Event()
                e = torch.cuda.Event()
                e.record(st)
                fake = torch.cuda.Stream()
                fake.wait_event(e)
                rt(st, N_GEO, N_AP, pieces, fake)
                ap_done.record(fake)
            torch.cuda._sleep(bin_cyc)
            if ap_done is not None:
                st.wait_event(ap_done)
            torch.cuda._sleep(rest_cyc)
            rt(st, 0, N_GEO, pieces, st)  # geometry down and back up

    for kind in ("base", "current", "pieces 1", "pieces 2", "pieces 4", "pieces 8"):
        for mode in ("eager", "graph"):
            if mode == "eager":
                run = lambda i: step(kind, i == 0)
            else:
                g0, g1 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
                torch.cuda.synchronize()
                with torch.cuda.graph(g0, stream=st):
                    step(kind, True)
                with torch.cuda.graph(g1, stream=st):
                    step(kind, False)
                run = lambda i: (g0 if i == 0 else g1).replay()
            for i in range(5):
                run(i)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            K = 100
            for i in range(K):
                run(i)
            torch.cuda.synchronize()
            print(f"{kind:10s} {mode:5s} {(time.perf_counter() - t0) / K * 1e3:.3f} ms/step", flush=True)


if __name__ == "__main__":
    main()
