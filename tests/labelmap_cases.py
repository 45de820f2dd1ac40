"""Label maps for the validate_label_map parity tests (valid, with unused ids,
with split regions), shared by the oracle (CPU) and device (GPU) tests."""
import numpy as np

from structure_cases import blob_labelmap, grid_labelmap, random_labelmap


def cases():
    rng = np.random.default_rng(2024)
    out = [
        ("ok_2x2", 2, 2, np.array([0, 0, 1, 1], np.uint32)),        # graph_test.cpp:161-166
        ("gap", 2, 1, np.array([0, 2], np.uint32)),                 # :168-172
        ("split", 3, 1, np.array([0, 1, 0], np.uint32)),            # :174-178
        ("diagonal", 2, 2, np.array([0, 1, 1, 0], np.uint32)),      # :180-184
        ("single", 5, 3, np.zeros(15, np.uint32)),
        ("huge_id", 3, 1, np.array([0, 1, 4_000_000_000], np.uint32)),
        ("one_pixel", 1, 1, np.array([0], np.uint32)),
    ]
    for i, (w, h, b) in enumerate(((7, 5, 2), (33, 17, 4), (64, 64, 8), (100, 37, 3))):
        reg = grid_labelmap(rng, w, h, b)[3]
        out.append((f"grid_{w}x{h}_{b}", w, h, reg))
        # relabel by a permutation: still valid
        perm = rng.permutation(int(reg.max()) + 1).astype(np.uint32)
        out.append((f"perm_{w}x{h}_{b}", w, h, perm[reg]))
        # drop one id (merge two neighbours' ids shifts the rest): unused id
        hole = reg.copy()
        hole[hole == hole.max()] += 1
        out.append((f"hole_{w}x{h}_{b}", w, h, hole))
        # split a region: give two distant pixels of different regions the same id
        split = reg.copy()
        split[-1] = split[0]
        out.append((f"split_{w}x{h}_{b}", w, h, split))
    for seed in range(6):
        w, h = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        R = max(1, min(w * h, int(rng.integers(1, 12))))
        out.append((f"random_{seed}", w, h,
                    random_labelmap(np.random.default_rng(seed), w, h, R)[3]))
        out.append((f"blob_{seed}", w, h, blob_labelmap(np.random.default_rng(seed), w, h)[3]))
    return out
