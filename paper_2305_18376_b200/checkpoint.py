"""Stream-state checkpoints in the reference's format (stream.py:409-540,
``STATE_FORMAT_VERSION`` 1).

Files are interchangeable with ``p2stream.save_state`` / ``load_state``:

* ``.json`` -- one document; floats written with Python's shortest exact
  repr, so a round trip is bit-exact.  Keys and their order match the
  reference, so the same state produces the same bytes.
* ``.npz`` -- raw float64 arrays ``w v c d f g``, one ``u_<i>`` per slice (in
  ``slice_ids`` order), optional ``smin_<i>`` / ``smax_<i>`` column stats, and
  a JSON ``meta`` blob stored as uint8.

The state lives on the GPU; saving reads it back once (each U-history block
is copied to the host once), loading builds a device-resident
:class:`~paper_2305_18376_b200.stream.StreamState`.
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .tensor import ColumnStats

STATE_FORMAT_VERSION = 1
_KIND = "stream-state"


def _bad_suffix(path: Path):
    return ValueError(f"unsupported checkpoint suffix {path.suffix!r} (use .json or .npz)")


def _stats_json(stats: ColumnStats | None):
    if stats is None:
        return None
    return {"minimum": {k: v.tolist() for k, v in stats.minimum.items()},
            "maximum": {k: v.tolist() for k, v in stats.maximum.items()}}


def save_state(state, path, column_stats: ColumnStats | None = None) -> None:
    """Write ``state`` (and optional normalisation stats) to ``.json`` / ``.npz``."""
    path = Path(path)
    ids = list(state.slice_ids)
    W, V, C, D, F, G = state.W, state.V, state.C, state.D, state.F, state.G
    if path.suffix == ".json":
        doc = {
            "format_version": STATE_FORMAT_VERSION,
            "kind": _KIND,
            "forgetting": state.forgetting,
            "update_index": state.update_index,
            "passes": state.passes,
            "rank": state.rank,
            "slice_ids": ids,
            "u": {sid: state.u_matrix(sid).tolist() for sid in ids},
            "w": W.tolist(),
            "v": V.tolist(),
            "helpers": {"c": {sid: C[k].tolist() for k, sid in enumerate(ids)},
                        "d": {sid: D[k].tolist() for k, sid in enumerate(ids)},
                        "f": F.tolist(),
                        "g": G.tolist()},
            "column_stats": _stats_json(column_stats),
        }
        path.write_text(json.dumps(doc))
        return
    if path.suffix == ".npz":
        arrays = {"w": W, "v": V, "c": C, "d": D, "f": F, "g": G}
        arrays.update({f"u_{i}": state.u_matrix(sid) for i, sid in enumerate(ids)})
        stats_ids = None
        if column_stats is not None:
            stats_ids = sorted(column_stats.minimum)
            for i, sid in enumerate(stats_ids):
                arrays[f"smin_{i}"] = column_stats.minimum[sid]
                arrays[f"smax_{i}"] = column_stats.maximum[sid]
        meta = {"format_version": STATE_FORMAT_VERSION, "kind": _KIND, "forgetting": state.forgetting,
                "update_index": state.update_index, "passes": state.passes, "slice_ids": ids,
                "stats_ids": stats_ids}
        arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
        np.savez(path, **arrays)
        return
    raise _bad_suffix(path)


def _check_version(found, path):
    if found != STATE_FORMAT_VERSION:
        raise ValueError(f"unsupported checkpoint format in {path}")


def load_state(path, device=None):
    """Read a checkpoint -> ``(StreamState on the GPU, ColumnStats | None)``."""
    from .stream import StreamState

    path = Path(path)
    f64 = lambda a: np.asarray(a, dtype=float)  # noqa: E731
    if path.suffix == ".json":
        doc = json.loads(path.read_text())
        _check_version(doc.get("format_version"), path)
        ids = list(doc["slice_ids"])
        h = doc["helpers"]
        state = StreamState(ids, {sid: [f64(doc["u"][sid])] for sid in ids}, f64(doc["w"]), f64(doc["v"]),
                            f64([h["c"][sid] for sid in ids]), f64([h["d"][sid] for sid in ids]),
                            f64(h["f"]), f64(h["g"]), float(doc["forgetting"]),
                            update_index=int(doc["update_index"]), passes=int(doc.get("passes", 1)),
                            device=device)
        raw = doc.get("column_stats")
        stats = None
        if raw is not None:
            stats = ColumnStats({k: f64(v) for k, v in raw["minimum"].items()},
                                {k: f64(v) for k, v in raw["maximum"].items()})
        return state, stats
    if path.suffix == ".npz":
        with np.load(path) as z:
            meta = json.loads(bytes(z["meta"]).decode())
            _check_version(meta.get("format_version"), path)
            ids = list(meta["slice_ids"])
            state = StreamState(ids, {sid: [z[f"u_{i}"]] for i, sid in enumerate(ids)}, z["w"], z["v"],
                                z["c"], z["d"], z["f"], z["g"], float(meta["forgetting"]),
                                update_index=int(meta["update_index"]), passes=int(meta.get("passes", 1)),
                                device=device)
            stats = None
            if meta.get("stats_ids") is not None:
                sids = list(meta["stats_ids"])
                stats = ColumnStats({sid: z[f"smin_{i}"] for i, sid in enumerate(sids)},
                                    {sid: z[f"smax_{i}"] for i, sid in enumerate(sids)})
        return state, stats
    raise _bad_suffix(path)
