"""Mesh (PLY/OBJ) and trajectory I/O for the session front end.

Host-side loading, run once per session; behaviour follows
texelfuse/meshio.py (load_mesh :25-47, load_trajectory :268-306): PLY
ascii / binary little- and big-endian with arbitrary vertex properties and
list faces, OBJ with fan triangulation, degenerate triangles dropped, and
DataError (naming the path) for unreadable or malformed files.
"""

import struct

import numpy as np

from .errors import DataError
from .geometry import CameraFrame, Intrinsics, Mesh

_PLY = {"char": "i1", "int8": "i1", "uchar": "u1", "uint8": "u1", "short": "i2", "int16": "i2",
        "ushort": "u2", "uint16": "u2", "int": "i4", "int32": "i4", "uint": "u4", "uint32": "u4",
        "float": "f4", "float32": "f4", "double": "f8", "float64": "f8"}


def _fan(faces):
    tris = []
    for f in faces:
        for k in range(1, len(f) - 1):
            tris.append((f[0], f[k], f[k + 1]))
    return np.asarray(tris, dtype=np.int64).reshape(-1, 3)


def _ply_header(fh, path):
    if fh.readline().strip() != b"ply":
        raise DataError("%s: not a PLY file" % path)
    fmt, elements = None, []
    while True:
        line = fh.readline()
        if not line:
            raise DataError("%s: unexpected end of PLY header" % path)
        tok = line.decode("ascii", "replace").split()
        if not tok or tok[0] == "comment":
            continue
        if tok[0] == "format":
            fmt = tok[1]
        elif tok[0] == "element":
            elements.append([tok[1], int(tok[2]), []])
        elif tok[0] == "property":
            if not elements:
                raise DataError("%s: property before element" % path)
            elements[-1][2].append(("list", tok[2], tok[3], tok[4]) if tok[1] == "list" else (tok[2], tok[1]))
        elif tok[0] == "end_header":
            break
    if fmt is None:
        raise DataError("%s: PLY header has no format line" % path)
    return fmt, elements


def _xyz_cols(props, path):
    names = [p[0] for p in props]
    for axis in "xyz":
        if axis not in names:
            raise DataError("%s: vertex element lacks %s property" % (path, axis))
    return [names.index(a) for a in "xyz"]


def _read_ply(path):
    with open(path, "rb") as fh:
        fmt, elements = _ply_header(fh, path)
        verts, faces = np.zeros((0, 3)), []
        if fmt == "ascii":
            for name, count, props in elements:
                if name == "vertex":
                    cols = _xyz_cols(props, path)
                    verts = np.empty((count, 3))
                    for i in range(count):
                        vals = fh.readline().split()
                        verts[i] = [float(vals[c]) for c in cols]
                elif name == "face":
                    for _ in range(count):
                        vals = fh.readline().split()
                        faces.append([int(v) for v in vals[1:1 + int(vals[0])]])
                else:
                    for _ in range(count):
                        fh.readline()
            return verts, faces
        if fmt not in ("binary_little_endian", "binary_big_endian"):
            raise DataError("%s: unsupported PLY format %r" % (path, fmt))
        e = "<" if fmt == "binary_little_endian" else ">"
        for name, count, props in elements:
            if not any(p[0] == "list" for p in props):
                dt = np.dtype([("f%d" % i, e + _PLY[p[1]]) for i, p in enumerate(props)])
                raw = fh.read(dt.itemsize * count)
                if len(raw) != dt.itemsize * count:
                    raise DataError("%s: truncated %s data" % (path, name))
                rec = np.frombuffer(raw, dtype=dt, count=count)
                if name == "vertex":
                    cols = _xyz_cols(props, path)
                    verts = np.stack([rec["f%d" % c].astype(np.float64) for c in cols], axis=1)
                continue
            for _ in range(count):
                face = None
                for p in props:
                    if p[0] == "list":
                        cdt, idt = np.dtype(e + _PLY[p[1]]), np.dtype(e + _PLY[p[2]])
                        b = fh.read(cdt.itemsize)
                        if len(b) != cdt.itemsize:
                            raise DataError("%s: truncated %s data" % (path, name))
                        n = int(np.frombuffer(b, cdt)[0])
                        b = fh.read(idt.itemsize * n)
                        if len(b) != idt.itemsize * n:
                            raise DataError("%s: truncated %s data" % (path, name))
                        if face is None:
                            face = np.frombuffer(b, idt, n).astype(np.int64).tolist()
                    else:
                        sz = np.dtype(_PLY[p[1]]).itemsize
                        if len(fh.read(sz)) != sz:
                            raise DataError("%s: truncated %s data" % (path, name))
                if name == "face":
                    faces.append(face or [])
        return verts, faces


def _read_obj(path):
    verts, faces = [], []
    with open(path, "r", encoding="utf-8", errors="replace") as fh:
        for ln, line in enumerate(fh, 1):
            tok = line.split()
            if not tok:
                continue
            try:
                if tok[0] == "v":
                    verts.append([float(t) for t in tok[1:4]])
                elif tok[0] == "f":
                    idx = []
                    for t in tok[1:]:
                        i = int(t.split("/")[0])
                        idx.append(i - 1 if i > 0 else len(verts) + i)
                    faces.append(idx)
            except ValueError as exc:
                raise DataError("%s:%d: %s" % (path, ln, exc)) from exc
    return np.asarray(verts, dtype=np.float64).reshape(-1, 3), faces


def load_mesh(path):
    """PLY or OBJ → Mesh with degenerate triangles dropped (meshio.py:25-47)."""
    path = str(path)
    try:
        with open(path, "rb") as fh:
            head = fh.read(4)
    except OSError as exc:
        raise DataError("cannot read mesh file %s: %s" % (path, exc)) from exc
    verts, faces = _read_ply(path) if head[:3] == b"ply" else _read_obj(path)
    if not len(verts):
        raise DataError("mesh %s has no vertices" % path)
    mesh = Mesh.from_arrays(verts, _fan(faces))
    if mesh.num_triangles == 0:
        raise DataError("mesh %s has no usable triangles" % path)
    return mesh


def save_ply(path, mesh, face_colors=None, binary=True):
    """Write float32 vertices and uchar-counted int faces (meshio.py:224-257)."""
    nv, nf = mesh.num_vertices, mesh.num_triangles
    hdr = ["ply", "format binary_little_endian 1.0" if binary else "format ascii 1.0",
           "element vertex %d" % nv, "property float x", "property float y", "property float z",
           "element face %d" % nf, "property list uchar int vertex_indices"]
    if face_colors is not None:
        face_colors = np.asarray(face_colors, dtype=np.uint8).reshape(nf, 3)
        hdr += ["property uchar red", "property uchar green", "property uchar blue"]
    hdr.append("end_header")
    v32 = mesh.vertices.astype("<f4")
    with open(path, "wb") as fh:
        fh.write(("\n".join(hdr) + "\n").encode("ascii"))
        if binary:
            fh.write(v32.tobytes())
            for i in range(nf):
                fh.write(struct.pack("<B3i", 3, *map(int, mesh.triangles[i])))
                if face_colors is not None:
                    fh.write(struct.pack("<3B", *map(int, face_colors[i])))
        else:
            for v in v32:
                fh.write(("%g %g %g\n" % tuple(v)).encode("ascii"))
            for i in range(nf):
                line = "3 %d %d %d" % tuple(mesh.triangles[i])
                if face_colors is not None:
                    line += " %d %d %d" % tuple(face_colors[i])
                fh.write((line + "\n").encode("ascii"))


def load_trajectory(path):
    """One camera per line: id fx fy cx cy w h then [R|t] row-major; sorted by id
    (meshio.py:268-306)."""
    try:
        with open(path, "r") as fh:
            lines = fh.read().splitlines()
    except OSError as exc:
        raise DataError("cannot read trajectory %s: %s" % (path, exc)) from exc
    frames, seen = [], set()
    for ln, raw in enumerate(lines, 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        vals = line.split()
        if len(vals) != 19:
            raise DataError("%s:%d: expected 19 fields, got %d" % (path, ln, len(vals)))
        try:
            fid = int(vals[0])
            nums = [float(v) for v in vals[1:]]
        except ValueError as exc:
            raise DataError("%s:%d: %s" % (path, ln, exc)) from exc
        if fid in seen:
            raise DataError("%s:%d: duplicate frame id %d" % (path, ln, fid))
        seen.add(fid)
        m = np.asarray(nums[6:], dtype=np.float64).reshape(3, 4)
        intr = Intrinsics(fx=nums[0], fy=nums[1], cx=nums[2], cy=nums[3], width=int(nums[4]), height=int(nums[5]))
        frames.append(CameraFrame(frame_id=fid, intrinsics=intr, rotation=m[:, :3], translation=m[:, 3]))
    if not frames:
        raise DataError("trajectory %s contains no frames" % path)
    frames.sort(key=lambda f: f.frame_id)
    return frames


def save_trajectory(path, frames):
    with open(path, "w") as fh:
        fh.write("# frame_id fx fy cx cy width height  r00 r01 r02 tx  r10 r11 r12 ty  r20 r21 r22 tz\n")
        for f in frames:
            mat = np.column_stack([f.rotation, f.translation]).reshape(-1)
            nums = [f.fx, f.fy, f.cx, f.cy, float(f.width), float(f.height), *mat]
            fh.write("%d %s\n" % (f.frame_id, " ".join("%.17g" % x for x in nums)))
