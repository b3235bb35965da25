"""numpy model of the x-slab exchange protocol (test infrastructure; the product runs it in C kernels:
csrc/fields.cu xplanes_pack / xplanes_unpack, csrc/sort.cu pack_migrants / unpack_migrants).

Arrays are a slab's whole-x-extent arrays: index i <-> global node x0 + i - G, owned [G, G + L).
"""

import numpy as np

G = 3


def pack_planes(arrays, which, L):
    """(to_left, to_right) messages of one slab (include/b200pic.h: which 0 J, 1 all E/B ghosts, 2 the
    planes maxwell_slab leaves stale)."""
    if which == 0:
        return (np.concatenate([a[0:2 * G + 1].ravel() for a in arrays]),
                np.concatenate([a[L:L + 2 * G + 1].ravel() for a in arrays]))
    if which == 1:
        blk = lambda a, i0, n: np.concatenate([a[i0:i0 + n], np.zeros_like(a[:G + 1 - n])]).ravel()
        return (np.concatenate([a[G:2 * G + 1].ravel() for a in arrays]),
                np.concatenate([blk(a, L, G) for a in arrays]))
    blk = lambda a, i0, n: np.concatenate([a[i0:i0 + n], np.zeros_like(a[:2 - n])]).ravel()
    return (np.concatenate([a[G + 2:G + 4].ravel() for a in arrays]),
            np.concatenate([blk(a, L, 1) for a in arrays]))


def unpack_planes(arrays, which, L, from_left, from_right):
    plane = arrays[0][0].size
    if which == 0:
        n = (2 * G + 1) * plane
        for k, a in enumerate(arrays):
            a[0:2 * G + 1] += from_left[k * n:(k + 1) * n].reshape(a[0:2 * G + 1].shape)
            a[L:L + 2 * G + 1] += from_right[k * n:(k + 1) * n].reshape(a[L:L + 2 * G + 1].shape)
        return
    np_ = G + 1 if which == 1 else 2
    nl = G if which == 1 else 1
    r0 = L + G if which == 1 else L + G + 2
    n = np_ * plane
    for k, a in enumerate(arrays):
        a[0:nl] = from_left[k * n:k * n + nl * plane].reshape(a[0:nl].shape)
        a[r0:L + 2 * G + 1] = from_right[k * n:(k + 1) * n].reshape(a[r0:L + 2 * G + 1].shape)


def pack_migrants(outgoing, cap):
    """outgoing: per species (left [8, n_l], right [8, n_r]) -> (to_left, to_right) float64 messages:
    int64 counts[S] (as raw bits), then per species [8][cap]."""
    S = len(outgoing)
    msgs = []
    for d in range(2):
        m = np.zeros(S + S * 8 * cap)
        for s, pair in enumerate(outgoing):
            blk = pair[d]
            m[s] = np.array([blk.shape[1]], np.int64).view(np.float64)[0]
            m[S + s * 8 * cap:S + (s + 1) * 8 * cap].reshape(8, cap)[:, :blk.shape[1]] = blk
        msgs.append(m)
    return msgs[0], msgs[1]


def unpack_migrants(msg, n_species, cap):
    out = []
    for s in range(n_species):
        cnt = int(msg[s:s + 1].view(np.int64)[0])
        blk = msg[n_species + s * 8 * cap:n_species + (s + 1) * 8 * cap].reshape(8, cap)
        out.append(blk[:, :min(cnt, cap)].copy())
    return out
