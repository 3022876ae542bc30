"""Engine timeline: `run` on the GPU box (writes gpurun_out/<tag>.npz), `show` here.

usage: python tools/timeline.py run TAG n nu ell eps kmax [kcap]
       python tools/timeline.py show gpurun_out/TAG.npz
"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
NAMES = ["fill", "aca", "tapp", "potrf", "trsm", "rapp", "seg", "proj", "prr", "phwp", "phwr", "nop"]


def run(tag, n, nu, ell, eps, kmax, kcap=0, nugget=1e-6):
    import torch
    import synth
    import paper_1709_08625_b200 as H
    s = synth.uniform_points(n, 1005)
    T = H.Tree(torch.from_numpy(s).cuda())
    Z = torch.from_numpy(synth.xi(n, 2005)).cuda()
    th = (1.0, ell, nu, nugget)
    r = H.eval_loglik(T, th, Z, eps, kmax, kcap)      # warm-up (allocations)
    path = f"/tmp/{tag}.bin"
    os.environ["HCOV_TIMELINE"] = path
    torch.cuda.synchronize()
    import time
    H.prof_control(True, True)
    t0 = time.time()
    r = H.eval_loglik(T, th, Z, eps, kmax, kcap)
    torch.cuda.synchronize()
    wall = time.time() - t0
    pr = H.prof_read()
    H.prof_control(False, True)
    print("phases ms:", {k: round(v, 1) for k, v in pr["phase_ms"].items()}, "flop:", pr["flop"], flush=True)
    print("phases by class:", pr["phase_cls_ms"], flush=True)
    del os.environ["HCOV_TIMELINE"]
    tl = np.fromfile(path, dtype=np.uint64).reshape(-1, 3)
    off, sc = T.succ()
    b = T.blocks()
    rm = (T.info()["n_pad"] >> b[b[:, 3] == 1][:, 0].astype(np.int64))
    out = f"/tmp/{tag}.npz"
    np.savez_compressed(out, tl=tl, tasks=T.tasks(), off=off, succ=sc, wall=wall, rm=rm,
                        result=np.array([r["loglik"], r["status"], r["max_rank"]]))
    print(tag, "wall", wall, r, flush=True)
    import contextlib
    import io
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        show(out)
    open(f"gpurun_out/{tag}.txt", "w").write(buf.getvalue())
    print(buf.getvalue())


def show(path):
    d = np.load(path)
    tl, tasks, off, sc = d["tl"].astype(np.int64), d["tasks"], d["off"], d["succ"]
    ty = tasks[:, 0]
    ran = tl[:, 1] > 0
    t0 = tl[ran, 0].min()
    st = np.where(ran, tl[:, 0] - t0, 0)
    en = np.where(ran, tl[:, 1] - t0, 0)
    dur = en - st
    print(f"wall {float(d['wall']):.3f}s  engine span {en.max()/1e9:.3f}s  result {d['result']}")
    print(f"{'type':6s} {'count':>8s} {'busy_s':>9s} {'mean_us':>9s} {'max_us':>9s}")
    for k, nm in enumerate(NAMES):
        m = (ty == k) & ran
        if m.any():
            print(f"{nm:6s} {m.sum():8d} {dur[m].sum()/1e9:9.3f} {dur[m].mean()/1e3:9.1f} {dur[m].max()/1e3:9.1f}")
    # predecessors via succ CSR
    n = len(ty)
    src = np.repeat(np.arange(n), np.diff(off))
    # finish time of NOPs = max of their preds' finish (completed inline)
    fin = en.copy()
    order = np.argsort(np.arange(n))  # tasks are in topological order
    preds = [[] for _ in range(n)]
    for a, b in zip(src, sc):
        preds[b].append(a)
    for t in range(n):
        if ty[t] == 11:
            fin[t] = max((fin[p] for p in preds[t]), default=0)
    # walk back the critical chain from the last-finishing task
    t = int(np.argmax(fin))
    chain = []
    while True:
        chain.append(t)
        if not preds[t]:
            break
        t = max(preds[t], key=lambda p: fin[p])
    chain = chain[::-1]
    busy = {}
    wait = 0
    prev_fin = 0
    for t in chain:
        if ty[t] == 11:
            continue
        busy[NAMES[ty[t]]] = busy.get(NAMES[ty[t]], 0) + dur[t]
        wait += max(0, st[t] - prev_fin)
        prev_fin = en[t]
    print(f"critical chain: {len([t for t in chain if ty[t] != 11])} tasks, span {fin[chain[-1]]/1e9:.3f}s, "
          f"busy {sum(busy.values())/1e9:.3f}s, queue/launch gaps {wait/1e9:.3f}s")
    print("  busy by type (s):", {k: round(v / 1e9, 4) for k, v in sorted(busy.items(), key=lambda x: -x[1])})
    # top 10 longest tasks on the chain
    cc = sorted([t for t in chain if ty[t] != 11], key=lambda t: -dur[t])[:10]
    rm = d["rm"] if "rm" in d else None

    def msize(t):
        return int(rm[tasks[t, 2]]) if rm is not None and ty[t] in (1, 5) else 0
    print("  longest on chain (type, m, ms):", [(NAMES[ty[t]], msize(t), round(dur[t] / 1e6, 3)) for t in cc])
    comp = {}
    for t in chain:
        if ty[t] == 11:
            continue
        key = f"{NAMES[ty[t]]}{msize(t) or ''}" + ("f" if ty[t] == 5 and tasks[t, 5] == 1 else "")
        cnt, tot = comp.get(key, (0, 0))
        comp[key] = (cnt + 1, tot + dur[t])
    # how the chain moves: critical predecessor of each chain rapp (same block's previous chunk or other)
    rch = [t for t in chain if ty[t] == 5]
    chain_nn = [t for t in chain if ty[t] != 11]
    if rch:
        same = sum(1 for a, b in zip(chain_nn[:-1], chain_nn[1:])
                   if ty[a] == 5 and ty[b] == 5 and tasks[a, 2] == tasks[b, 2])
        blocks = len(set(int(tasks[t, 2]) for t in rch))
        runs, cur = [], 1
        for a, b in zip(rch[:-1], rch[1:]):
            if tasks[a, 2] == tasks[b, 2]:
                cur += 1
            else:
                runs.append(cur)
                cur = 1
        runs.append(cur)
        print(f"  chain rapp: {len(rch)} tasks over {blocks} blocks; same-block chunk->chunk edges {same}; "
              f"run lengths mean {np.mean(runs):.1f} max {max(runs)}")
        preds_ty = {}
        for a, b in zip(chain_nn[:-1], chain_nn[1:]):
            if ty[b] == 5:
                k = NAMES[ty[a]] + ("(same)" if ty[a] == 5 and tasks[a, 2] == tasks[b, 2] else "")
                preds_ty[k] = preds_ty.get(k, 0) + 1
        print("  critical predecessor of chain rapps:", preds_ty)
    print("  chain composition (type+m[f=final chunk]: count, total ms):",
          {k: (v[0], round(v[1] / 1e6, 1)) for k, v in sorted(comp.items(), key=lambda x: -x[1][1])})
    if rm is not None:
        for k in (1, 5):
            m = (ty == k) & ran
            if m.any():
                sizes = rm[tasks[m, 2]]
                print(f"  {NAMES[k]} by block size (m: count, mean ms, max ms):",
                      {int(z): (int((sizes == z).sum()), round(dur[m][sizes == z].mean() / 1e6, 2),
                                round(dur[m][sizes == z].max() / 1e6, 2)) for z in np.unique(sizes)})


if __name__ == "__main__":
    if sys.argv[1] == "run":
        a = sys.argv[2:]
        run(a[0], int(a[1]), float(a[2]), float(a[3]), float(a[4]), int(a[5]), int(a[6]) if len(a) > 6 else 0,
            float(a[7]) if len(a) > 7 else 1e-6)
    else:
        show(sys.argv[2])
