"""Replay of recorded node states: readers for the
reference's snapshot and trajectory files, so benchmarks and tests can blend
with node graphs a SLAM run recorded instead of synthetic lattices.

    snapshot  (snapshot.hpp:17-44, write_snapshot): one JSON object per file,
              {"hex_spacing", "nodes": [{"anchor", "position", "scale",
              "dq": [w, z, dx, dy], "variance"}], "keyframes", "feature_tracks"}
    trajectory (snapshot.hpp:80-124, TrajectoryWriter / load_trajectory): one
              JSON line per frame, {"frame", "status", "new_anchors",
              "positions"}; anchors accumulate over the lines.

A snapshot gives exactly blend_frame's node inputs (anchors = graph.anchors(),
warps = graph.warps() as (scale, w, z, dx, dy), mosaic.hpp:196) plus the node
positions and variances (the inputs of variance_field,
Engine::blended_variance_at slam.hpp:703-714)."""
from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import List, Union

import numpy as np


@dataclass
class Snapshot:
    hex_spacing: float
    anchors: np.ndarray      # (n, 2) reference-frame anchors
    warps: np.ndarray        # (n, 5) WarpFunction {scale, w, z, dx, dy}
    positions: np.ndarray    # (n, 2) current positions (warp(anchor))
    variances: np.ndarray    # (n,)
    tracks: np.ndarray       # (m, 3) feature tracks: x, y, variance
    keyframes: List[dict]


def _text(src: Union[str, bytes, Path]) -> str:
    if isinstance(src, bytes):
        return src.decode()
    if isinstance(src, Path) or (isinstance(src, str) and not src.lstrip().startswith(("{", "["))):
        return Path(src).read_text()
    return src


def read_snapshot(src) -> Snapshot:
    """write_snapshot's JSON (a path or the text) -> Snapshot."""
    d = json.loads(_text(src))
    nodes = d.get("nodes", [])
    n = len(nodes)
    anchors = np.zeros((n, 2))
    warps = np.zeros((n, 5))
    pos = np.zeros((n, 2))
    var = np.zeros(n)
    for i, nd in enumerate(nodes):
        anchors[i] = nd["anchor"]
        warps[i, 0] = nd["scale"]
        warps[i, 1:] = nd["dq"]
        pos[i] = nd["position"]
        var[i] = nd["variance"]
    tr = d.get("feature_tracks", [])
    tracks = np.array([[t["position"][0], t["position"][1], t["variance"]] for t in tr]).reshape(-1, 3)
    return Snapshot(float(d.get("hex_spacing", 0.0)), anchors, warps, pos, var, tracks, list(d.get("keyframes", [])))


@dataclass
class Trajectory:
    anchors: np.ndarray          # (n_total, 2) in insertion order
    positions: List[np.ndarray]  # per frame (n_t, 2)
    status: List[str]
    frames: List[int]


def read_trajectory(src) -> Trajectory:
    """load_trajectory (snapshot.hpp:107-124): TrajectoryWriter's JSON lines."""
    anchors, positions, status, frames = [], [], [], []
    for line in _text(src).splitlines():
        if not line.strip():
            continue
        j = json.loads(line)
        anchors.extend(j["new_anchors"])
        positions.append(np.array(j["positions"], np.float64).reshape(-1, 2))
        status.append(j["status"])
        frames.append(int(j.get("frame", len(frames))))
    return Trajectory(np.array(anchors, np.float64).reshape(-1, 2), positions, status, frames)
