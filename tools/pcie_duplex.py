"""Host link microbenchmark: pinned host <-> device copies on the copy engines,
each direction alone and both at once (the e2e leg of bench.py streams the
gradients in and the updated parameters out concurrently).  Prints one JSON
line per pattern: GB/s per direction and aggregate."""
import json
import sys

import torch


def main():
    gib = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    n = gib << 29                              # int16 elements: gib GiB
    h_in = torch.empty(n, dtype=torch.int16, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.int16, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.int16, device="cuda")
    d_out = torch.empty(n, dtype=torch.int16, device="cuda")
    h_in.fill_(1)
    d_out.fill_(2)
    s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
    nbytes = 2 * n
    chunks = 8

    def run(up, dn, reps=5):
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(s_up)
        e[2].record(s_dn)
        c = n // chunks
        for _ in range(reps):
            for k in range(chunks):
                if up:
                    with torch.cuda.stream(s_up):
                        d_in[k * c:(k + 1) * c].copy_(h_in[k * c:(k + 1) * c], non_blocking=True)
                if dn:
                    with torch.cuda.stream(s_dn):
                        h_out[k * c:(k + 1) * c].copy_(d_out[k * c:(k + 1) * c], non_blocking=True)
        e[1].record(s_up)
        e[3].record(s_dn)
        torch.cuda.synchronize()
        t_up = e[0].elapsed_time(e[1]) / 1e3 / reps
        t_dn = e[2].elapsed_time(e[3]) / 1e3 / reps
        t = max(t_up if up else 0.0, t_dn if dn else 0.0)
        out = {"pattern": ("h2d" if up else "") + ("+" if up and dn else "") + ("d2h" if dn else ""),
               "bytes_per_direction": nbytes}
        if up:
            out["h2d_GBps"] = round(nbytes / t_up / 1e9, 1)
        if dn:
            out["d2h_GBps"] = round(nbytes / t_dn / 1e9, 1)
        out["aggregate_GBps"] = round(nbytes * (int(up) + int(dn)) / t / 1e9, 1)
        return out

    run(True, True, 1)   # warm-up
    for up, dn in ((True, False), (False, True), (True, True)):
        print(json.dumps(run(up, dn)), flush=True)


if __name__ == "__main__":
    main()
