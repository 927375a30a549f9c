"""Train BASELINE c4's two OpInf ROMs with the CPU oracle (calls only oracle/) and write them out.

    python tools/gen_c4_rom.py            # ~15-30 min on 8 cores

Offline stage of Algorithm 2 with top-down training (remark:training P:L527-543, reading
R25): an O-SAM FOM-FOM-FOM run on 80^3 meshes per subdomain (oracle.opinf.train_coupled), 500 steps ->
501 snapshots per subdomain; POD r = 200, boundary POD by the 99.9999% energy rule, ridge OpInf lambda =
1e-8.  Writes

  var/c4_ops/<i>_<name>.npy      the full operators (Phi is 1.6M x 200 = 2.5 GB per ROM) for the oracle's
                                 own online run (tools/gen_golden_fullsize.py c4); not shipped to the GPU;
  cache/c4_rom_ops.npz           what the online library needs (~160 MB): Phi restricted to the free DOFs
                                 the Schwarz transfer reads from each ROM ("Phi restricted to the relevant
                                 boundary DoFs") with their row indices, Phi_dS, Kbar, Bbar, and the
                                 reduced IC u^0 = Phi^T u0[free], s0 = u0[Schwarz DOFs] computed
                                 by the oracle's ROM.init_state.

No value comes from the CUDA path.  `load_full_ops()` / `load_online_ops()` read them back.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import osam_inputs as I  # noqa: E402

FULL_DIR = os.path.join(ROOT, "var", "c4_ops")
ONLINE = os.path.join(ROOT, "cache", "c4_rom_ops.npz")
NAMES = ("Phi", "Phi_s", "Kbar", "Bbar", "sigma", "sigma_s")


def load_full_ops():
    ops = {}
    for i in (0, 2):
        d = {k: np.load(os.path.join(FULL_DIR, f"{i}_{k}.npy"), mmap_mode="r" if k == "Phi" else None) for k in NAMES}
        with open(os.path.join(FULL_DIR, f"{i}_meta.json")) as fh:
            d.update(json.load(fh))
        d["Phi"] = np.asarray(d["Phi"])
        ops[i] = d
    return ops


def rom_ops_id(ops):
    """Identity of one training run: sha256 over Kbar and Bbar of both ROMs (the noise modes beyond the snapshot
    rank differ from run to run, so golden data belongs to exactly one set of operators)."""
    import hashlib
    h = hashlib.sha256()
    for i in (0, 2):
        h.update(np.ascontiguousarray(ops[i]["Kbar"], dtype=np.float64).tobytes())
        h.update(np.ascontiguousarray(ops[i]["Bbar"], dtype=np.float64).tobytes())
    return h.hexdigest()


def load_online_ops(path=ONLINE):
    """{i: dict(phi_rows, Phi (rows subset), Phi_s, Kbar, Bbar, uh0, s0, n_free, r, r_b)} or None if absent."""
    if not os.path.exists(path):
        return None
    z = np.load(path)
    out = {}
    for i in (0, 2):
        out[i] = {k: z[f"{i}_{k}"] for k in ("phi_rows", "Phi", "Phi_s", "Kbar", "Bbar", "uh0", "s0", "n_free")}
        out[i]["r"] = out[i]["Kbar"].shape[0]
        out[i]["r_b"] = out[i]["Bbar"].shape[1]
    return out


def main():
    from oracle import opinf, schwarz

    cfg = I.config("c4")
    t0 = time.time()
    ops = opinf.train(cfg, I)
    t_train = time.time() - t0
    print(f"trained in {t_train:.0f}s", {i: (o["r"], o["r_b"]) for i, o in ops.items()}, flush=True)
    os.makedirs(FULL_DIR, exist_ok=True)
    for i, o in ops.items():
        for k in NAMES:
            np.save(os.path.join(FULL_DIR, f"{i}_{k}.npy"), np.asarray(o[k]))
        with open(os.path.join(FULL_DIR, f"{i}_meta.json"), "w") as fh:
            json.dump(dict(r=int(o["r"]), r_b=int(o["r_b"]), lam=float(o["lam"]), dt=float(o["dt"])), fh)
    models = schwarz.build_models(cfg, ops)
    data = {}
    meta = dict(script="tools/gen_c4_rom.py", train_seconds=round(t_train, 1), source="oracle only")
    for i, o in ops.items():
        m = models[i]
        rows = set()
        for j, mj in enumerate(models):
            for src, sel, nodes, w in (mj._proj or []):
                if src != i:
                    continue
                dofs = (3 * nodes.reshape(-1)[:, None] + np.arange(3)[None, :]).reshape(-1)
                r_ = m.free_row[dofs]
                rows.update(int(x) for x in r_[r_ >= 0])
        rows = np.array(sorted(rows), dtype=np.int64)
        st = m.init_state(I.initial_displacements(cfg, cfg["subdomains"][i]))
        data.update({f"{i}_phi_rows": rows, f"{i}_Phi": np.asfortranarray(o["Phi"][rows]),
                     f"{i}_Phi_s": np.asfortranarray(o["Phi_s"]), f"{i}_Kbar": o["Kbar"], f"{i}_Bbar": o["Bbar"],
                     f"{i}_uh0": st["uh"][0], f"{i}_s0": st["s"][0], f"{i}_n_free": np.array(len(m.free_dofs))})
        sig = np.asarray(o["sigma"])
        meta[str(i)] = dict(r=int(o["r"]), r_b=int(o["r_b"]), n_free=int(len(m.free_dofs)), lift_rows=int(len(rows)),
                            numerical_rank_1e13=int((sig > 1e-13 * sig[0]).sum()),
                            kbar_max_abs_imag_eig=float(np.abs(np.linalg.eigvals(o["Kbar"]).imag).max()))
        print(i, meta[str(i)], flush=True)
    os.makedirs(os.path.dirname(ONLINE), exist_ok=True)
    np.savez(ONLINE, **data)
    with open(os.path.join(FULL_DIR, "provenance.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("wrote", ONLINE, os.path.getsize(ONLINE) / 1e6, "MB", flush=True)


if __name__ == "__main__":
    main()
