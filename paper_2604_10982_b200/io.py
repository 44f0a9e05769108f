"""The reference's on-disk formats for the render path, in numpy:
scene checkpoints (.psimap, proj/src/io.cpp:386-494), raw planes (PSIPLANE, io.cpp:319-384)
and camera JSON (io.cpp:126-161). Byte-compatible with include/psimap_b200_io.hpp and the
reference (little-endian, the field order of save_checkpoint)."""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .panoptic import InstanceQuery
from .raster import Camera, SceneMap

CKPT_MAGIC = b"PSIMAPCK"
CKPT_VERSION = 1
RAW_MAGIC = b"PSIPLANE"


@dataclass
class Checkpoint:
    """Everything save_checkpoint writes: the scene, its vocabulary, the queries with their
    bookkeeping, and the attention weights (carried, not used by render)."""
    scene: SceneMap
    vocabulary: List[str] = field(default_factory=list)
    class_votes: List[List[int]] = field(default_factory=list)
    assign_count: List[int] = field(default_factory=list)
    attn_w: tuple = (np.zeros((0, 0)), np.zeros((0, 0)), np.zeros((0, 0)))  # w_q, w_k, w_v (C_ins x d)
    pos_enc_bands: int = 6
    pos_enc_base_freq: float = 0.5
    pos_enc_seed: int = 42


def save_checkpoint(path: str, ck: Checkpoint) -> None:
    sc = ck.scene
    n = len(sc)
    c_sem = sc.c_sem()
    f_ins = sc.f_ins if sc.f_ins is not None else np.zeros((n, 0))
    c_ins = f_ins.shape[1] if n else 0
    out = [CKPT_MAGIC, struct.pack("<II", CKPT_VERSION, len(ck.vocabulary))]
    for v in ck.vocabulary:
        b = v.encode()
        out.append(struct.pack("<I", len(b)) + b)
    out.append(struct.pack("<IIQ", c_sem, c_ins, n))
    if n:
        rows = np.concatenate([sc.surfels, sc.f_sem.reshape(n, c_sem), f_ins.reshape(n, c_ins)], axis=1)
        out.append(np.ascontiguousarray(rows, dtype="<f8").tobytes())
    out.append(struct.pack("<Q", len(sc.queries)))
    for i, q in enumerate(sc.queries):
        f = np.asarray(q.feature, dtype="<f8").reshape(-1)
        votes = ck.class_votes[i] if i < len(ck.class_votes) else []
        cnt = ck.assign_count[i] if i < len(ck.assign_count) else 0
        out.append(struct.pack("<I", f.size) + f.tobytes())
        out.append(np.asarray(q.mean, dtype="<f8").reshape(3).tobytes())
        out.append(np.asarray(q.cov, dtype="<f8").reshape(3, 3).T.reshape(9).tobytes())  # column-major
        out.append(struct.pack("<I", len(votes)) + struct.pack(f"<{len(votes)}q", *votes))
        out.append(struct.pack("<iqB", q.class_id, cnt, 1 if q.alive else 0))
    wq, wk, wv = ck.attn_w
    out.append(struct.pack("<II", wq.shape[0], wq.shape[1]))
    for m in (wq, wk, wv):
        out.append(np.asarray(m, dtype="<f8").T.reshape(-1).tobytes())  # MatX column-major
    out.append(struct.pack("<idQ", ck.pos_enc_bands, ck.pos_enc_base_freq, ck.pos_enc_seed))
    with open(path, "wb") as fh:
        fh.write(b"".join(out))


def load_checkpoint(path: str) -> Checkpoint:
    buf = open(path, "rb").read()
    pos = 0

    def take(fmt):
        nonlocal pos
        sz = struct.calcsize(fmt)
        if pos + sz > len(buf):
            raise RuntimeError("checkpoint: unexpected end of file")
        v = struct.unpack_from(fmt, buf, pos)
        pos += sz
        return v

    def doubles(k):
        nonlocal pos
        if pos + 8 * k > len(buf):
            raise RuntimeError("checkpoint: truncated surfel data")
        a = np.frombuffer(buf, dtype="<f8", count=k, offset=pos).astype(np.float64)
        pos += 8 * k
        return a

    if buf[:8] != CKPT_MAGIC:
        raise RuntimeError(f"bad checkpoint magic: {path}")
    pos = 8
    (version,) = take("<I")
    if version != CKPT_VERSION:
        raise RuntimeError(f"unsupported checkpoint version {version}")
    (nv,) = take("<I")
    vocab = []
    for _ in range(nv):
        (ln,) = take("<I")
        vocab.append(buf[pos:pos + ln].decode())
        pos += ln
    c_sem, c_ins, n = take("<IIQ")
    rows = doubles(n * (13 + c_sem + c_ins)).reshape(n, 13 + c_sem + c_ins)
    (nq,) = take("<Q")
    queries, votes, counts = [], [], []
    for _ in range(nq):
        (nf,) = take("<I")
        feat = doubles(nf)
        mean = doubles(3)
        cov = doubles(9).reshape(3, 3).T
        (nvt,) = take("<I")
        votes.append(list(take(f"<{nvt}q")) if nvt else [])
        cls, cnt, alive = take("<iqB")
        counts.append(cnt)
        queries.append(InstanceQuery(feature=feat, mean=mean, cov=cov, class_id=cls, alive=bool(alive)))
    r, c = take("<II")
    ws = tuple(doubles(r * c).reshape(c, r).T for _ in range(3))
    bands, freq, seed = take("<idQ")
    scene = SceneMap(rows[:, :13], rows[:, 13:13 + c_sem], rows[:, 13 + c_sem:] if c_ins else None, queries)
    return Checkpoint(scene, vocab, votes, counts, ws, bands, freq, seed)


def save_raw(path: str, plane: np.ndarray) -> None:
    """PSIPLANE: magic, W, H, C (u32), dtype 0 = f64 / 1 = i32, then HWC payload."""
    a = np.asarray(plane)
    h, w = a.shape[:2]
    c = a.shape[2] if a.ndim == 3 else 1
    dt = 1 if np.issubdtype(a.dtype, np.integer) else 0
    payload = a.astype("<i4" if dt else "<f8").tobytes()
    with open(path, "wb") as fh:
        fh.write(RAW_MAGIC + struct.pack("<IIII", w, h, c, dt) + payload)


def load_raw(path: str) -> np.ndarray:
    buf = open(path, "rb").read()
    if buf[:8] != RAW_MAGIC:
        raise RuntimeError(f"bad raw plane magic: {path}")
    w, h, c, dt = struct.unpack_from("<IIII", buf, 8)
    a = np.frombuffer(buf, dtype="<i4" if dt == 1 else "<f8", offset=24)
    if a.size != w * h * c:
        raise RuntimeError(f"truncated raw plane: {path}")
    return a.reshape(h, w, c).copy()


def camera_to_json(cam: Camera) -> str:
    c = cam.to_c()
    return json.dumps({"r_cw": list(c.r_cw), "t_cw": list(c.t_cw), "fx": c.fx, "fy": c.fy, "cx": c.cx, "cy": c.cy,
                       "width": c.width, "height": c.height, "near": c.near_clip, "far": c.far_clip},
                      indent=2, sort_keys=True)


def camera_from_json(text: str) -> Camera:
    j = json.loads(text)
    near, far = j.get("near", 0.01), j.get("far", 100.0)
    if "eye" in j:
        return Camera.look_at(tuple(j["eye"]), tuple(j["target"]), tuple(j.get("up", (0, 1, 0))), j["fx"], j["fy"],
                              int(j["width"]), int(j["height"]), near, far)
    r = np.asarray(j["r_cw"], dtype=np.float64).reshape(3, 3).T  # column-major in the file
    return Camera.make(r, np.asarray(j["t_cw"], dtype=np.float64), j["fx"], j["fy"], j["cx"], j["cy"],
                       int(j["width"]), int(j["height"]), near, far)
