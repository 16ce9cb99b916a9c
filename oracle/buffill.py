"""Alg. "Hit buffer filling" (§4) -- TEST INFRASTRUCTURE.

A line-by-line transcription of the paper's storeHit procedure, used to pin
the product's native implementation (paper_2412_11809_b200/csrc/buffill.h)
hit by hit.  Pure Python loops: small inputs only.

    constant b        maximum buffer size
    constant t_closing small interval added to the final boundary time
    constant b_t      hits that can arrive within t + t_closing
    global   toa_max  <- 0
    storeHit(hit, buffer, nextBuffer):
        if size(buffer) < b - b_t:            buffer += hit; toa_max = max(toa_max, toa(hit))
        elif toa(hit) < toa_max + t_closing:  buffer += hit
        else:                                 nextBuffer += hit
        if toa(hit) - toa_max > t + t_closing:
            sendToDevice(buffer); buffer <- nextBuffer

Readings (R20): nextBuffer starts empty again after a send; a sent
buffer's cut is C = toa_max + t_closing (every later hit of a t-ordered
stream has toa >= C); at the end of the stream the open
buffer is sent with cut C if nextBuffer holds hits, then nextBuffer with an
infinite cut (every cluster closed).
"""
from __future__ import annotations

import numpy as np

INF = (1 << 64) - 1


def buffill(hits, b: int, b_t: int, t: int, t_closing: int):
    """Returns (buffer_id uint32[n], cuts list[int]): the buffer each hit is
    sent in (in order of sending) and each sent buffer's cut."""
    toa = np.asarray(hits["toa"], dtype=np.uint64).tolist()
    n = len(toa)
    buffer_id = np.zeros(n, dtype=np.uint32)
    cuts = []
    toa_max = 0
    buffer, next_buffer = [], []
    for i in range(n):
        h = toa[i]
        if len(buffer) < b - b_t:
            buffer.append(i)
            toa_max = max(toa_max, h)
        elif h < toa_max + t_closing:
            buffer.append(i)
        else:
            next_buffer.append(i)
        if h > toa_max + t + t_closing:  # toa(hit) - toa_max > t + t_closing
            for j in buffer:
                buffer_id[j] = len(cuts)
            cuts.append(toa_max + t_closing)
            buffer, next_buffer = next_buffer, []
    # end of stream (reading R20)
    if next_buffer:
        for j in buffer:
            buffer_id[j] = len(cuts)
        cuts.append(toa_max + t_closing)
        buffer, next_buffer = next_buffer, []
    if buffer:
        for j in buffer:
            buffer_id[j] = len(cuts)
        cuts.append(INF)
    return buffer_id, cuts
