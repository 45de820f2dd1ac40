"""CPU restatement of the partitioned optimize schedule (csrc/partition.cu),
one rank per process over torch.distributed (gloo) -- TEST INFRASTRUCTURE.

Each rank runs the MAP kernels' arithmetic (numpy, the exact IEEE operation
order of label_energy, model.hpp:66-72, and of the slot-order hood fold,
engine.cpp:147-152) over only the vertices / series it owns, moves the halo
windows of parallel.halo_windows with isend/irecv, sums the unconverged-hood
counters with all_reduce and, per EM iteration, allgathers the leaf partials
of the last hood-energy row (each rank folds its own 1024-element leaves)
and runs the distributed M-step of partition.cu (label counts, head
fragments and owned-leaf partials allgathered -- never the labels, which are
gathered once at the end); the folds and the EM total are the C oracle's
(update_parameters, engine.cpp:193-223; dpp::reduce, kernels.hpp:124-139).
The result must equal the oracle's one-process optimize bit for bit, which
checks the partition plan and the exchange schedule independently of CUDA.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from oracle import C
from paper_1809_05018_b200.parallel import halo_windows


def _distributed_update(orc, mean_own, lab_own, mu, sigma, world, rank):
    """update_parameters (engine.cpp:193-223) distributed as in partition.cu
    (k_part_count .. k_part_unpack_partials): no rank sees the others'
    labels.  Every rank counts its own labels per label, the counts are
    allgathered; rank r's vertices are label l's segment [off_r, off_r + n_r)
    of the stable grouping x; a rank folds the 1024-element leaves that START
    in its segments, reading the later ranks' head fragments (their first
    elements up to the next leaf boundary, allgathered) where a leaf straddles;
    the owned-leaf partials are allgathered and every rank runs fold_tree per
    label -- sum pass, then the (x - mu)^2 pass."""
    M = len(mu)
    cnt = np.bincount(lab_own, minlength=M).astype(np.int64)
    allcnt = _allgather(cnt, M, world).reshape(world, M)
    n = allcnt.sum(axis=0)
    off = np.concatenate([np.zeros((1, M), np.int64), np.cumsum(allcnt, axis=0)])  # [q][l]
    seg = [mean_own[lab_own == l] for l in range(M)]  # (stable: vertex order)
    head_len = lambda o, c: min(c, (1024 - o % 1024) % 1024)  # noqa: E731
    heads = np.zeros(M * 1024)
    for l in range(M):
        h = head_len(int(off[rank][l]), int(cnt[l]))
        heads[l * 1024:l * 1024 + h] = seg[l][:h]
    all_heads = _allgather(heads, M * 1024, world).reshape(world, M, 1024)

    def owned(q, l):  # leaves j with off_q <= 1024 j < off_q + n_q
        o, c = int(off[q][l]), int(allcnt[q][l])
        first = (o + 1023) // 1024
        return range(first, (o + c + 1023) // 1024 if c else first)

    cap = (len(mean_own) + 1023) // 1024 + M + 1
    leaves_of = [(int(c) + 1023) // 1024 for c in n]
    mu, sigma = mu.copy(), sigma.copy()
    for sq in (False, True):
        own = np.zeros(cap)
        k = 0
        for l in range(M):
            for j in owned(rank, l):
                b = 1024 * j - int(off[rank][l])
                vals = list(seg[l][b:b + 1024])
                q = rank + 1
                while len(vals) < 1024 and 1024 * j + len(vals) < n[l] and q < world:
                    h = head_len(int(off[q][l]), int(allcnt[q][l]))
                    vals += list(all_heads[q, l, :h])[:1024 - len(vals)]
                    q += 1
                v = np.asarray(vals)
                if sq:
                    d = v - mu[l]
                    v = d * d
                own[k] = orc.fold_range(v)
                k += 1
        gathered = _allgather(own, cap, world).reshape(world, cap)
        for l in range(M):
            if n[l] == 0:
                continue  # empty labels keep their parameters (engine.cpp:209-211)
            parts = np.zeros(leaves_of[l])
            for q in range(world):
                base = sum(len(owned(q, ll)) for ll in range(l))
                for i, j in enumerate(owned(q, l)):
                    parts[j] = gathered[q][base + i]
            folded = orc.fold_tree(parts)
            if not sq:
                mu[l] = folded / float(n[l])
            else:
                sigma[l] = max(np.sqrt(folded / float(n[l])), 1e-3)
    return mu, sigma


def _exchange(arr, win, me, world):
    """Send my windows of arr to their destinations, receive the others' windows."""
    reqs = []
    for o in range(world):
        if o == me:
            continue
        lo, hi = int(win[me, o, 0]), int(win[me, o, 1])
        if lo <= hi:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(arr[lo:hi + 1])), o))
        lo, hi = int(win[o, me, 0]), int(win[o, me, 1])
        if lo <= hi:
            buf = torch.empty(hi - lo + 1, dtype=torch.from_numpy(arr[:1]).dtype)
            reqs.append((dist.irecv(buf, o), lo, hi, buf))
    for r in reqs:
        if isinstance(r, tuple):
            r[0].wait()
            arr[r[1]:r[2] + 1] = r[3].numpy()
        else:
            r.wait()


def _allgather(own, chunk, world):
    parts = [torch.empty(chunk, dtype=torch.from_numpy(own[:1]).dtype) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(own)))
    return np.concatenate([p.numpy() for p in parts])


def optimize_rank(graph, hoods, cfg, fixed_work=False):
    """One rank's share of the partitioned optimize; returns (labels, mu, sigma, totals, T)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    orc = C()
    off = np.asarray(graph.offsets, np.int64)
    nbr = np.asarray(graph.neighbors, np.int64)
    mean = np.asarray(graph.region_mean, np.float64)
    R = len(off) - 1
    h_off = np.asarray(hoods.offsets, np.int64)
    mem = np.asarray(hoods.members, np.int64)
    sizes = np.diff(h_off)
    s_off = np.concatenate([[0], np.cumsum(sizes[sizes > 0])]).astype(np.int64)
    s_first = h_off[:-1][sizes > 0]
    Hs = len(s_off) - 1
    # series members in slot order (empty hoods dropped, as reduce_by_key does)
    s_mem = np.concatenate([mem[a:a + n] for a, n in zip(s_first, sizes[sizes > 0])]) \
        if Hs else mem[:0]
    plan = halo_windows(off, nbr, s_off, s_mem, world)
    vb, ve = int(plan.vb[rank]), int(plan.vb[rank + 1])
    hb, he = int(plan.hb[rank]), int(plan.hb[rank + 1])
    cover = np.zeros(R, bool)
    cover[mem] = True
    M, L, tol, beta = cfg.num_labels, cfg.convergence_window, cfg.convergence_tol, cfg.beta
    mu, sigma, lab0 = orc.init_random(M, R, cfg.rng_seed, allow_multilabel=M != 2)
    lab = [lab0.astype(np.int64), lab0.astype(np.int64).copy()]
    minE = np.zeros(R)
    own_v = np.arange(vb, ve)
    deg = off[vb + 1:ve + 1] - off[vb:ve]
    v_rep = np.repeat(np.arange(ve - vb), deg)
    v_nbr = nbr[off[vb]:off[ve]]
    own_sz = s_off[hb + 1:he + 1] - s_off[hb:he]
    own_start = s_off[hb:he]
    cur = 0
    totals, em_T, em_hist = [], [], []
    for em in range(cfg.em_max_iters):
        _, two_var, log_sigma = orc.label_terms(mu, sigma)
        hist = []
        T = 0
        for t in range(cfg.map_max_iters):
            lin, lout = lab[(cur + t) & 1], lab[(cur + t + 1) & 1]
            # vertex pass over the owned range (engine.cpp:74-191 fused)
            x = mean[vb:ve]
            best = None
            arg = np.zeros(ve - vb, np.int64)
            for l in range(M):
                disc = np.zeros(ve - vb, np.int64)
                np.add.at(disc, v_rep, (lin[v_nbr] != l).astype(np.int64))
                d = x - mu[l]
                e = ((d * d) / two_var[l] + log_sigma[l]) + beta * disc.astype(np.float64)
                if best is None:
                    best = e
                else:
                    take = e < best
                    best = np.where(take, e, best)
                    arg = np.where(take, l, arg)
            minE[vb:ve] = best
            lout[vb:ve] = np.where(cover[vb:ve], arg, lin[vb:ve])
            _exchange(lout, plan.lab_win, rank, world)
            _exchange(minE, plan.min_win, rank, world)
            # hood pass over the owned series: left fold in slot order
            sums = np.zeros(he - hb)
            if he > hb:
                sums = minE[s_mem[own_start]].copy()
                for j in range(1, int(own_sz.max())):
                    m = j < own_sz
                    sums[m] = sums[m] + minE[s_mem[own_start[m] + j]]
            hist.append(sums)
            flags = orc.check_convergence(np.array(hist), L, tol) if he > hb else \
                np.zeros(0, np.uint8)
            unconv = torch.tensor([int((flags == 0).sum())], dtype=torch.int64)
            dist.all_reduce(unconv)
            T = t + 1
            if not fixed_work and int(unconv.item()) == 0:
                break
        cur = (cur + T) & 1
        # the rank's hood-series leaves (its series range starts on a leaf
        # boundary) folded locally; only the leaf partials are exchanged
        chunk_l = plan.chunk_h // 1024
        own_parts = np.zeros(chunk_l)
        row_own = hist[-1]
        for i in range((he - hb + 1023) // 1024):
            own_parts[i] = orc.fold_range(row_own[i * 1024:(i + 1) * 1024])
        parts = _allgather(own_parts, chunk_l, world)[:(Hs + 1023) // 1024]
        mu, sigma = _distributed_update(orc, mean[vb:ve], lab[cur][vb:ve], mu, sigma, world,
                                        rank)
        total = orc.fold_tree(parts) if len(parts) else 0.0
        totals.append(total)
        em_T.append(T)
        em_hist.append(total)
        conv = len(em_hist) >= L + 1 and all(
            abs(total - em_hist[-1 - i]) < tol for i in range(1, L + 1))
        if conv and not fixed_work:
            break
    # the labels are gathered once, after the EM loop
    own_lab = np.zeros(plan.chunk_v, np.int64)
    own_lab[:ve - vb] = lab[cur][vb:ve]
    full_lab = _allgather(own_lab, plan.chunk_v, world)[:R]
    return full_lab.astype(np.uint32), mu, sigma, totals, em_T
