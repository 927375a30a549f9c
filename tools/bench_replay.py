"""Throughput of the batched subdomain-local replay (osam_opinf_replay, NEXT-4): n_models candidate
ROMs x K training steps in one call, inputs resident on the device; CUDA-event timing around the call
(it includes the per-call allocations, the operator transpose, the replay kernel and the argmin).
Seeded synthetic operators of the sizes of the BASELINE workloads (c2: r = 20, K = 400; c5: r = 400,
K = 2001), 40 models (the paper's grid size)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_20687_b200 import osam  # noqa: E402


def case(r, r_b, K, B, order=1, reps=5):
    rng = np.random.default_rng(r)
    w = np.linspace(100.0, 15000.0, r)
    Q = np.linalg.qr(rng.standard_normal((r, r)))[0]
    nf = (r * (r + 1) // 2 if order >= 2 else 0)
    base = np.concatenate([-(Q * w ** 2) @ Q.T, rng.standard_normal((r, r_b)), 1e-3 * rng.standard_normal((r, nf))], 1)
    dev = "cuda:0"
    Ocm = torch.from_numpy(np.ascontiguousarray(np.stack([base * (1 + 0.01 * k) for k in range(B)]).transpose(0, 2, 1))).to(dev)
    Ub = torch.from_numpy(np.asfortranarray(1e-3 * rng.standard_normal((r, K))).T.copy()).to(dev)
    Gh = torch.from_numpy((1e-3 * rng.standard_normal((r_b, K))).T.copy()).to(dev)
    err = torch.empty(B, dtype=torch.float64, device=dev)
    d = osam.osam_replay_desc(r, r_b, order, B, K, 1e-4, Ocm.data_ptr(), Ub.data_ptr(), Gh.data_ptr(), None)
    best = osam.C.c_int32()
    s = torch.cuda.current_stream()
    L = osam.lib()
    for _ in range(2):
        osam._check(L.osam_opinf_replay(osam.C.byref(d), osam.C.c_void_p(err.data_ptr()), osam.C.byref(best), None,
                                        osam.C.c_void_p(s.cuda_stream)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        osam._check(L.osam_opinf_replay(osam.C.byref(d), osam.C.c_void_p(err.data_ptr()), osam.C.byref(best), None,
                                        osam.C.c_void_p(s.cuda_stream)))
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return dict(r=r, r_b=r_b, K=K, models=B, order=order, ms_per_call=ms,
                model_steps_per_s=B * (K - 1) / (ms * 1e-3), us_per_step=ms * 1e3 / (K - 1))


if __name__ == "__main__":
    for args in ((20, 43, 400, 40), (200, 40, 2001, 40), (400, 40, 2001, 40), (20, 43, 400, 40, 2)):
        print(json.dumps(case(*args)))
