"""Panoptic layer over the render path: the query-to-surfel
label assignment (psimap::assign_labels, proj/src/panoptic.cpp:36-91) and the panoptic
prediction planes (psimap::render_panoptic, proj/src/metrics.cpp:339-369), both on the GPU
through the C-ABI (psm_assign_labels, psm_render_panoptic)."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np


@dataclass
class InstanceQuery:
    """psimap::InstanceQuery (core_types.hpp:76-84): feature (C_ins), a 3D Gaussian
    (mean, SPD cov) and the class id voted for it."""
    feature: np.ndarray
    mean: np.ndarray = field(default_factory=lambda: np.zeros(3))
    cov: np.ndarray = field(default_factory=lambda: np.eye(3))
    class_id: int = -1
    alive: bool = True


@dataclass
class PanopticRender:
    """psimap::PanopticRender (metrics.hpp:70-78): int32 (H, W, 1) planes, -1 = void."""
    ids: np.ndarray
    classes: np.ndarray
    sem_classes: np.ndarray


def pack_queries(queries: Sequence[InstanceQuery], c_ins: int) -> Tuple[np.ndarray, ...]:
    """Flat arrays for the C-ABI: feat (Q, C_ins), mean (Q, 3), cov (Q, 9) column-major, alive,
    class ids."""
    q = len(queries)
    feat = np.zeros((q, c_ins))
    mean = np.zeros((q, 3))
    cov = np.zeros((q, 9))
    alive = np.zeros(q, np.int32)
    cls = np.full(q, -1, np.int32)
    for i, qu in enumerate(queries):
        f = np.asarray(qu.feature, dtype=np.float64).reshape(-1)
        if f.shape[0] != c_ins:
            raise ValueError("feature_similarity: dimension mismatch")  # panoptic.cpp:12-14
        feat[i] = f
        mean[i] = np.asarray(qu.mean, dtype=np.float64).reshape(3)
        cov[i] = np.asarray(qu.cov, dtype=np.float64).reshape(3, 3).T.reshape(9)  # column-major
        alive[i] = 1 if qu.alive else 0
        cls[i] = qu.class_id
    return feat, mean, cov, alive, cls


def panoptic_epilogue(alpha_acc: np.ndarray, ins_argmax: np.ndarray, sem_feat: np.ndarray,
                      query_class: Sequence[int]) -> PanopticRender:
    """The per-pixel body of render_panoptic (metrics.cpp:349-366) over render planes:
    alpha < 0.5 is void; id = label argmax; class = the id's query class; semantic class =
    first max of the feature plane."""
    h, w = alpha_acc.shape[:2]
    gate = alpha_acc[..., 0] >= 0.5
    ids = np.where(gate, ins_argmax[..., 0], -1).astype(np.int32)
    qc = np.asarray(query_class, dtype=np.int32)
    classes = np.full((h, w), -1, np.int32)
    ok = gate & (ids >= 0) & (ids < len(qc))
    classes[ok] = qc[ids[ok]]
    sem = np.full((h, w), -1, np.int32)
    if sem_feat.shape[-1] > 0:
        sem[gate] = np.argmax(sem_feat[gate], axis=-1)  # first max, as the strict > scan
    return PanopticRender(ids[..., None], classes[..., None], sem[..., None])


def street_queries(n_queries: int, c_ins: int = 8, seed: int = 11) -> List[InstanceQuery]:
    """Synthetic queries for the street workload (the reference's make_street_scene has
    none): Gaussians spread over the street volume (x in [-4, 4], y in [-3, 1.5], z in
    [2, 38]) with random unit-scale features and classes 0..7."""
    rng = np.random.default_rng(seed)
    out = []
    for q in range(n_queries):
        mean = np.array([rng.uniform(-4, 4), rng.uniform(-3, 1.5), rng.uniform(2, 38)])
        s = np.diag([rng.uniform(1, 3), rng.uniform(1, 3), rng.uniform(2, 6)]) ** 2
        out.append(InstanceQuery(feature=0.3 * rng.standard_normal(c_ins), mean=mean, cov=s, class_id=q % 8))
    return out
