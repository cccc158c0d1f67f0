"""ASCII MSH 2.2 import/export for the assembly's element connectivity (host-side I/O).

Restates the reference reader (import_msh, mesh.cpp:129-288; write_msh, :290-310) and extends it
to the 3D meshes this build assembles:
  * header must be "2.2 0 8"; $Nodes before $Elements; node ids reindexed to dense 0-based ids in
    file order; duplicate / unknown node ids, short sections and missing end markers are
    MshParseError (same messages);
  * kind "quad4" (the reference): 4-node quads (type 3) are kept, points and lines ignored,
    other surface elements skipped with a warning, volume elements are an error;
  * kind "tet4" (type 4) or "hex8" (type 5, Gmsh local order = meshgen's): that volume type is
    kept, points/lines/surfaces are ignored, other volume types are an error. kind "auto" picks
    the first retained type found (quad4 when there is no volume element).
Hex27 is not read or written: Gmsh's 27-node order differs from meshgen's lexicographic order.
"""
from __future__ import annotations

import numpy as np

IGNORED = {15, 1, 8, 26, 27}                      # points and lines (mesh.cpp:94-96)
SURFACE = {2, 9, 10, 16, 20, 21, 22, 23, 24, 25, 3}  # triangles, quads (mesh.cpp:100-114)
VOLUME_TYPES = {"tet4": 4, "hex8": 5}
NODES_OF = {3: 4, 4: 4, 5: 8}


class MshParseError(ValueError):
    """fea::MshParseError (types.hpp:36-38)."""


def _lines(text: str):
    for line in text.splitlines():
        yield line.rstrip("\r")


def import_msh(text: str, kind: str = "quad4"):
    """-> (conn (E, npe) int64, n_nodes, coords (n_nodes, 3), warnings, kind)."""
    it = _lines(text)

    def next_content():
        for line in it:
            if line.strip():
                return line
        raise MshParseError("unexpected end of file")

    node_ids: dict[int, int] = {}
    coords = []
    elements = []
    warnings = []
    seen_format = seen_nodes = seen_elements = False
    skipped = 0
    want = None if kind == "auto" else (3 if kind == "quad4" else VOLUME_TYPES[kind])
    for line in it:
        if not line or line[0] != "$":
            continue
        section = line[1:]
        if section == "MeshFormat":
            f = next_content().split()
            if len(f) < 3 or f[0] != "2.2" or f[1] != "0" or f[2] != "8":
                raise MshParseError('unsupported mesh format header (expected "2.2 0 8")')
            if next_content() != "$EndMeshFormat":
                raise MshParseError("missing $EndMeshFormat")
            seen_format = True
        elif section == "Nodes":
            if not seen_format:
                raise MshParseError("$Nodes before $MeshFormat")
            try:
                count = int(next_content().split()[0])
            except (ValueError, IndexError):
                raise MshParseError("malformed node count") from None
            if count < 0:
                raise MshParseError("malformed node count")
            for _ in range(count):
                nl = next_content()
                if nl == "$EndNodes":
                    raise MshParseError("node section ended before declared count")
                f = nl.split()
                try:
                    nid, x, y, z = int(f[0]), float(f[1]), float(f[2]), float(f[3])
                except (ValueError, IndexError):
                    raise MshParseError("malformed node line") from None
                if nid in node_ids:
                    raise MshParseError("duplicate node id")
                node_ids[nid] = len(coords)
                coords.append((x, y, z))
            if next_content() != "$EndNodes":
                raise MshParseError("missing $EndNodes")
            seen_nodes = True
        elif section == "Elements":
            if not seen_nodes:
                raise MshParseError("$Elements before $Nodes")
            try:
                count = int(next_content().split()[0])
            except (ValueError, IndexError):
                raise MshParseError("malformed element count") from None
            if count < 0:
                raise MshParseError("malformed element count")
            for _ in range(count):
                el = next_content()
                if el == "$EndElements":
                    raise MshParseError("element section ended before declared count")
                f = el.split()
                try:
                    etype, ntags = int(f[1]), int(f[2])
                except (ValueError, IndexError):
                    raise MshParseError("malformed element line") from None
                if ntags < 0 or len(f) < 3 + ntags:
                    raise MshParseError("malformed element tags")
                if want is None and etype in NODES_OF and (etype != 3 or kind == "auto"):
                    want = etype
                if etype == want:
                    refs = f[3 + ntags:3 + ntags + NODES_OF[etype]]
                    if len(refs) != NODES_OF[etype]:
                        raise MshParseError("malformed element connectivity")
                    try:
                        elements.append([node_ids[int(r)] for r in refs])
                    except KeyError:
                        raise MshParseError("element references unknown node id") from None
                    except ValueError:
                        raise MshParseError("malformed element connectivity") from None
                elif etype in IGNORED:
                    pass
                elif etype in SURFACE:
                    if want in (None, 3):
                        skipped += 1
                else:
                    raise MshParseError(f"mesh contains non-{'quad' if want in (None, 3) else kind} "
                                        f"volume or unknown element type {etype}")
            if next_content() != "$EndElements":
                raise MshParseError("missing $EndElements")
            seen_elements = True
        else:
            end = "$End" + section
            for line2 in it:
                if line2 == end:
                    break
            else:
                raise MshParseError("unterminated section " + section)
    if not (seen_format and seen_nodes and seen_elements):
        raise MshParseError("file lacks $MeshFormat, $Nodes or $Elements")
    if skipped:
        warnings.append(f"skipped {skipped} non-quad surface element(s)")
    kinds = {3: "quad4", 4: "tet4", 5: "hex8"}
    npe = NODES_OF.get(want, 4)
    conn = np.array(elements, dtype=np.int64).reshape(-1, npe)
    return conn, len(coords), np.array(coords, dtype=np.float64).reshape(-1, 3), warnings, kinds.get(want, "quad4")


def write_msh(conn, coords, kind: str, os) -> None:
    """write_msh (mesh.cpp:290-310) for quad4 / tet4 / hex8: 1-based ids, tags "2 0 1"."""
    etype = {"quad4": 3, "tet4": 4, "hex8": 5}[kind]
    coords = np.asarray(coords, dtype=np.float64)
    os.write("$MeshFormat\n2.2 0 8\n$EndMeshFormat\n")
    os.write(f"$Nodes\n{len(coords)}\n")
    for i, c in enumerate(coords):
        z = c[2] if len(c) > 2 else 0.0
        os.write(f"{i + 1} {c[0]:.17g} {c[1]:.17g} {z:.17g}\n")
    os.write("$EndNodes\n")
    os.write(f"$Elements\n{len(conn)}\n")
    for e, el in enumerate(np.asarray(conn)):
        os.write(f"{e + 1} {etype} 2 0 1 " + " ".join(str(int(v) + 1) for v in el) + "\n")
    os.write("$EndElements\n")


def structured_coords(kind: str, n: int) -> np.ndarray:
    """Node coordinates matching meshgen's numbering (unit square / cube)."""
    h = 1.0 / n
    ax = np.arange(n + 1) * h
    if kind == "quad4":
        y, x = np.meshgrid(ax, ax, indexing="ij")
        return np.stack([x.ravel(), y.ravel(), np.zeros(x.size)], axis=1)
    z, y, x = np.meshgrid(ax, ax, ax, indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)
