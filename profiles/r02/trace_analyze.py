"""Per-layer in-graph timeline of the model decode step from an LKV_XP_TRACE replay
(profiles/model_step_time.py --trace FILE.npy with the experiment build).

Every CTA of the step's GEMVs, per-layer attention and combine recorded (entry, griddepcontrol.wait
released, exit) on %globaltimer.  Launches of a kind are split by CTA count; per layer (1 .. L-2,
averaged), each launch's first entry / first and last wait release / last exit relative to the
layer's QKV first entry, in microseconds."""
import sys

import numpy as np

NAMES = {0: "qkv", 16: "qkv", 100: "attn", 101: "comb", 17: "wo|down", 2: "gate/up", 3: "lm_head"}


def main(path):
    r = np.load(path)
    kind = r["kind"] % 1000
    keep = ~((r["kind"] >= 1000) & (kind == 101))  # combine: only the y = 0 CTAs
    r, kind = r[keep], kind[keep]
    launches = {}
    for k in np.unique(kind):
        rk = r[kind == k]
        rk = rk[np.argsort(rk["t0"], kind="stable")]
        n_l = {0: 32, 16: 32, 100: 32, 101: 32, 17: 64, 2: 32, 3: 1}[int(k)]
        per = len(rk) // n_l
        launches[int(k)] = [rk[i * per:(i + 1) * per] for i in range(n_l)]
        print(f"{NAMES[int(k)]:8s} launches {n_l} CTAs/launch {per} (records {len(rk)})")
    seq = []
    for l in range(32):
        wo, down = launches[17][2 * l], launches[17][2 * l + 1]
        qkv = launches[0] if 0 in launches else launches[16]  # stream-K or split-K cluster
        seq.append([("qkv", qkv[l]), ("attn", launches[100][l]), ("comb", launches[101][l]), ("wo", wo),
                    ("gate/up", launches[2][l]), ("down", down)])
    t_start = seq[0][0][1]["t0"].min()
    t_end = launches[3][0]["t5"].max()
    print(f"step (first qkv entry -> lm_head exit): {(t_end - t_start) / 1e3:.1f} us")
    rows = {}
    for l in range(1, 31):
        base = seq[l][0][1]["t0"].min()
        prev_end = seq[l - 1][5][1]["t5"].max()
        rows.setdefault("prev down end", []).append((prev_end - base) / 1e3)
        for name, x in seq[l]:
            rows.setdefault(name, []).append(
                [(x["t0"].min() - base) / 1e3, (x["t1"].min() - base) / 1e3, (x["t1"].max() - base) / 1e3,
                 (np.median(x["t5"]) - base) / 1e3, (x["t5"].max() - base) / 1e3])
        rows.setdefault("layer", []).append((seq[l + 1][0][1]["t0"].min() - base) / 1e3)
    print("per layer (mean over layers 1..30), us from the layer's first QKV CTA entry")
    print(f"  previous down last exit {np.mean(rows['prev down end']):7.2f}")
    print(f"  {'kernel':8s} {'entry0':>7s} {'wait0':>7s} {'waitN':>7s} {'exitMed':>7s} {'exitN':>7s}")
    for name in ("qkv", "attn", "comb", "wo", "gate/up", "down"):
        m = np.mean(np.array(rows[name]), axis=0)
        print(f"  {name:8s} " + " ".join(f"{v:7.2f}" for v in m))
    print(f"  next layer's qkv entry {np.mean(rows['layer']):7.2f}")
    # inner phases (fields t2..t4, 0 = not recorded): median / max over CTAs, relative to wait release
    print("inner phases, us after the launch's first wait release: median / max over CTAs")
    print("  stream-K (qkv, gate/up): t2 first group's unit loop done, t3 fix-up arrival, t4 fix-up summed")
    print("  split (wo, down): t2 consume done, t3 cluster barrier, t4 DSMEM reduce done (rank 0)")
    names = ("t2", "t3", "t4", "t5")
    for name in ("qkv", "wo", "gate/up", "down"):
        acc = {k: [] for k in names}
        for l in range(1, 31):
            x = dict(seq[l])[name]
            w0 = x["t1"].min()
            for k in names:
                v = x[k][x[k] > 0]
                if len(v):
                    acc[k].append([(np.median(v) - w0) / 1e3, (v.max() - w0) / 1e3])
        print(f"  {name:8s} " + "  ".join(
            f"{k} {np.mean(np.array(acc[k])[:, 0]):6.2f}/{np.mean(np.array(acc[k])[:, 1]):6.2f}" for k in names if acc[k]))


if __name__ == "__main__":
    main(sys.argv[1])
