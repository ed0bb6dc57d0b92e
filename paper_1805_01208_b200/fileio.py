"""METIS graph files, coordinate files and partition files, read and written on the GPU
(the reference's fileio.py:70-278).

Same functions, arguments, results and error messages as the reference.  The file bytes
are uploaded once; csrc/textio.cu tokenizes them (lines, tokens, every token converted
where it starts: integers exactly, decimal reals correctly rounded by Eisel-Lemire) and
assembles the CSR arrays; csrc/graphs.cu checks duplicates, symmetry and edge-weight
symmetry with the radix sort, as the reference does with argsort.

What stays on the host, by design:
  * the header line (one line) and the MESSAGE of an error: the device finds the first
    line the reference would reject, the host re-reads that one line with the
    reference's own per-line logic (restated in `_vertex_line`) to word the error;
  * tokens outside the plain decimal grammar (``nan``, ``1_000``, more than 19
    significant digits, an inconclusive Eisel-Lemire product): Python's int()/float()
    or numpy's converter decides them, token by token, and the values are patched in.
    A file written by the reference's writers has none;
  * `write_metis_graph` / `write_coords` (fileio.py:199-216, :240-243): the generator
    side, not on the partition path.
Bytes that are not printable ASCII, tab, CR or LF are rejected (the reference decodes
ASCII and also breaks lines at form feeds etc.; such files are not supported here).
"""

from __future__ import annotations

import io
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .graph import (CHK_ASYM, CHK_EW_ASYM, CHK_PARALLEL, GeometricGraph, check_structure)
from .types import Partition

__all__ = [
    "MetisParseError", "load_metis_graph", "write_metis_graph", "load_coords", "write_coords",
    "read_partition", "write_partition",
]

TOK_INT, TOK_REAL, TOK_PERCENT, TOK_SUSPECT = 0, 1, 2, 3


class MetisParseError(ValueError):
    """Raised for malformed graph, coordinate, or partition files."""


# ---------------------------------------------------------------- sources and sinks
def _read_bytes(source) -> np.ndarray:
    """The raw bytes of a path, text stream or byte stream (fileio.py:35-53)."""
    if isinstance(source, (str, Path)):
        path = os.fspath(source)
        if os.path.getsize(path) >= (64 << 20):
            # large files: map the page cache; the staging ring's host threads copy it
            # straight into pinned chunks (no intermediate buffer)
            return np.memmap(path, dtype=np.uint8, mode="r")
        return np.fromfile(path, dtype=np.uint8)
    data = source.read()
    if isinstance(data, str):
        data = data.encode("ascii")
    return np.frombuffer(bytearray(data), dtype=np.uint8)


def _write_bytes(sink, data: bytes) -> None:
    if isinstance(sink, (str, Path)):
        with open(sink, "wb") as f:
            f.write(data)
    elif isinstance(sink, io.TextIOBase) or hasattr(sink, "encoding"):
        sink.write(data.decode("ascii"))
    else:
        sink.write(data)


# ---------------------------------------------------------------- device tokenizer
@dataclass
class _Tokens:
    host: np.ndarray          # the file bytes
    n_lines: int
    n_tokens: int
    line_off: object          # device int64 (n_lines + 1)
    line_tok0: object         # device int64 (n_lines + 1)
    tok_val: object           # device int64 (n_tokens)
    tok_kind: object          # device uint8 (n_tokens)

    def line_text(self, line: int) -> str:
        return self.lines_text([line])[line]

    def lines_text(self, lines) -> dict:
        """{line: its text} for a batch of line numbers (one device read for all)."""
        import torch

        if not len(lines):
            return {}
        idx = torch.as_tensor(sorted(set(int(v) for v in lines)), dtype=torch.int64,
                              device=self.line_off.device)
        lo = self.line_off[idx].cpu().tolist()
        hi = self.line_off[idx + 1].cpu().tolist()
        return {int(l): bytes(self.host[a:b]).decode("ascii").rstrip("\r\n")
                for l, a, b in zip(idx.cpu().tolist(), lo, hi)}


def _tokenize(buf: np.ndarray, comment_char: int) -> _Tokens:
    import torch

    from . import _native as N
    from . import staging

    n = int(buf.shape[0])
    sh = torch.cuda.current_stream().cuda_stream
    text = torch.empty(n, dtype=torch.uint8, device="cuda")
    staging.h2d_into(text, buf)
    wsb = N.size_query("gp_text_index_workspace_bytes", n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    counts = torch.empty(3, dtype=torch.int64, device="cuda")
    N.call("gp_text_index", text.data_ptr(), n, comment_char, counts.data_ptr(), ws.data_ptr(),
           wsb, sh)
    n_lines, n_tokens, n_odd = (int(v) for v in counts.cpu().tolist())
    if n_odd:
        pos = int(np.flatnonzero((buf >= 0x7f) | ((buf < 0x20) & (buf != 9) & (buf != 10)
                                                  & (buf != 13)))[0])
        if buf[pos] >= 0x80:
            raise UnicodeDecodeError("ascii", bytes(buf[pos:pos + 1]), 0, 1,
                                     f"ordinal not in range(128) at byte {pos}")
        raise ValueError(f"unsupported control character 0x{int(buf[pos]):02x} at byte {pos}")
    line_off = torch.empty(n_lines + 1, dtype=torch.int64, device="cuda")
    line_tok0 = torch.empty(n_lines + 1, dtype=torch.int64, device="cuda")
    tok_val = torch.empty(max(n_tokens, 1), dtype=torch.int64, device="cuda")
    tok_kind = torch.empty(max(n_tokens, 1), dtype=torch.uint8, device="cuda")
    N.call("gp_text_tokens", text.data_ptr(), n, comment_char, ws.data_ptr(), n_lines, n_tokens,
           line_off.data_ptr(), line_tok0.data_ptr(), tok_val.data_ptr(), tok_kind.data_ptr(), sh)
    return _Tokens(buf, n_lines, n_tokens, line_off, line_tok0, tok_val, tok_kind)


def _to_host(t) -> np.ndarray:
    """A device tensor as a numpy array, through the pinned staging ring."""
    from . import staging

    out = np.empty(tuple(t.shape), dtype={"torch.int64": np.int64, "torch.float64": np.float64,
                                          "torch.uint8": np.uint8}[str(t.dtype)])
    if out.size:
        staging.d2h_into(out, t.contiguous())
    return out


# ---------------------------------------------------------------- METIS graph
def _fail(lineno, msg):
    raise MetisParseError(f"line {lineno}: {msg}")


def _weight(tok, lineno, what):
    try:
        w = float(tok)
    except ValueError:
        _fail(lineno, f"non-numeric {what} {tok!r}")
    if not w > 0 or not np.isfinite(w):
        _fail(lineno, f"{what} must be strictly positive, got {tok!r}")
    return w


def _header(text: str, lineno: int):
    """(n, m, has_vwgt, has_ewgt) of the header line (fileio.py:95-122)."""
    parts = text.split()
    if len(parts) < 2 or len(parts) > 4:
        _fail(lineno, f"header must be 'n m [fmt [ncon]]', got {text!r}")
    try:
        n, m = int(parts[0]), int(parts[1])
    except ValueError:
        _fail(lineno, "non-numeric vertex or edge count")
    if n < 1 or m < 0:
        _fail(lineno, f"bad sizes n={n} m={m}")
    fmt = parts[2] if len(parts) >= 3 else "0"
    if not fmt.isdigit():
        _fail(lineno, f"non-numeric fmt {fmt!r}")
    has_vsize, has_vwgt, has_ewgt = (c == "1" for c in fmt.zfill(3))
    if has_vsize:
        _fail(lineno, "vertex sizes (fmt 1xx) are not supported")
    ncon = 1
    if len(parts) == 4:
        try:
            ncon = int(parts[3])
        except ValueError:
            _fail(lineno, f"non-numeric ncon {parts[3]!r}")
    if has_vwgt and ncon != 1:
        _fail(lineno, f"only one vertex weight per vertex is supported, got ncon={ncon}")
    return n, m, has_vwgt, has_ewgt


def _vertex_line(text: str, lineno: int, u: int, n: int, has_vwgt: bool, has_ewgt: bool):
    """One vertex line read the reference's way (fileio.py:131-160): raises its error, or
    returns (vertex weight, 0-based neighbor ids, edge weights or None)."""
    toks = text.split()
    vw, pos = 1.0, 0
    if has_vwgt:
        if not toks:
            _fail(lineno, "missing vertex weight")
        vw, pos = _weight(toks[0], lineno, "vertex weight"), 1
    rest = toks[pos:]
    if has_ewgt and len(rest) % 2:
        _fail(lineno, "dangling neighbor without edge weight")
    ids = rest[0::2] if has_ewgt else rest
    nbrs = []
    for tok in ids:
        try:
            v = int(tok)
        except ValueError:
            _fail(lineno, f"non-numeric neighbor id {tok!r}")
        if v < 1 or v > n:
            _fail(lineno, f"neighbor id {v} out of range 1..{n}")
        if v == u + 1:
            _fail(lineno, f"self loop at vertex {u + 1}")
        nbrs.append(v - 1)
    if len(set(nbrs)) != len(nbrs):
        _fail(lineno, f"duplicate neighbor in adjacency list of vertex {u + 1}")
    ews = [_weight(t, lineno, "edge weight") for t in rest[1::2]] if has_ewgt else None
    return vw, nbrs, ews


def load_metis_graph(graph_source, coord_source=None) -> GeometricGraph:
    """Read a METIS graph file plus a coordinate file into a graph (fileio.py:70-196).

    ``coord_source`` None gives every vertex coordinate (0, 0).  Raises
    :class:`MetisParseError` naming the offending line for malformed headers,
    non-numeric tokens, ids out of range, line-count mismatches and asymmetric
    adjacency, exactly as the reference does.
    """
    import torch

    from . import _native as N

    buf = _read_bytes(graph_source)
    if buf.shape[0] == 0:
        raise MetisParseError("line 1: missing header")
    tk = _tokenize(buf, 0)
    sh = torch.cuda.current_stream().cuda_stream
    dev = "cuda"
    wsb = N.size_query("gp_metis_workspace_bytes", tk.n_lines)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    body_line = torch.empty(tk.n_lines, dtype=torch.int64, device=dev)
    info = torch.empty(3, dtype=torch.int64, device=dev)
    N.call("gp_metis_lines", tk.line_tok0.data_ptr(), tk.tok_kind.data_ptr(), tk.n_lines,
           body_line.data_ptr(), tk.n_lines, info.data_ptr(), ws.data_ptr(), wsb, sh)
    n_plain, header_line, last_used = (int(v) for v in info.cpu().tolist())
    if n_plain == 0:
        raise MetisParseError("line 1: missing header")
    header_no = header_line + 1
    n, m, has_vwgt, has_ewgt = _header(tk.line_text(header_line), header_no)
    # trailing all-whitespace lines beyond the declared vertex count are ignored
    n_body = n_plain - 1
    if n_body > n:
        n_body = max(n, last_used)
    if n_body != n:
        raise MetisParseError(
            f"line {header_no}: header declares {n} vertices but file has {n_body} vertex lines")
    if n >= 2 ** 31 - 1:
        raise MetisParseError(f"line {header_no}: more than 2^31 vertices are not supported")

    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    flags = torch.empty(n, dtype=torch.uint8, device=dev)
    N.call("gp_metis_offsets", tk.line_tok0.data_ptr(), body_line.data_ptr(), n, int(has_vwgt),
           int(has_ewgt), offsets.data_ptr(), flags.data_ptr(), ws.data_ptr(), wsb, sh)
    nnz = int(offsets[n].item())
    neighbors = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)[:nnz]
    ew = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)[:nnz] if has_ewgt else None
    vw = torch.empty(n, dtype=torch.float64, device=dev) if has_vwgt else None
    N.call("gp_metis_fill", tk.line_tok0.data_ptr(), body_line.data_ptr(), tk.tok_val.data_ptr(),
           tk.tok_kind.data_ptr(), n, int(has_vwgt), int(has_ewgt), offsets.data_ptr(),
           neighbors.data_ptr(), None if ew is None else ew.data_ptr(),
           None if vw is None else vw.data_ptr(), flags.data_ptr(), sh)

    def structure():
        if nnz >= 2 ** 31:
            raise MetisParseError(
                f"line {header_no}: more than 2^31 adjacency entries are not supported")
        return check_structure(offsets, neighbors, ew, n, vertex_flags=flags)

    chk, missing = structure()
    flagged = torch.nonzero(flags).flatten()
    if flagged.numel():
        # the host words the error of the first rejected line; a flagged line that Python
        # accepts (exotic but valid tokens) is patched with Python's values
        lines = body_line[flagged].cpu().tolist()
        texts = tk.lines_text(lines)
        starts = offsets[flagged].cpu().tolist()
        ends = offsets[flagged + 1].cpu().tolist()
        p_pos, p_nb, p_ew, p_u, p_vw = [], [], [], [], []
        for u, line, o0, o1 in zip(flagged.cpu().tolist(), lines, starts, ends):
            w, nb, ews = _vertex_line(texts[line], line + 1, u, n, has_vwgt, has_ewgt)
            if len(nb) != o1 - o0:
                raise RuntimeError(f"line {line + 1}: tokenizer and host disagree on the degree")
            p_pos.extend(range(o0, o1))
            p_nb.extend(nb)
            if has_ewgt:
                p_ew.extend(ews)
            p_u.append(u)
            p_vw.append(w)
        # every flagged line was accepted by Python: patch its values in
        if p_pos:
            pos = torch.tensor(p_pos, dtype=torch.int64, device=dev)
            neighbors[pos] = torch.tensor(p_nb, dtype=torch.int64, device=dev)
            if has_ewgt:
                ew[pos] = torch.tensor(p_ew, dtype=torch.float64, device=dev)
        if has_vwgt:
            vw[torch.tensor(p_u, dtype=torch.int64, device=dev)] = \
                torch.tensor(p_vw, dtype=torch.float64, device=dev)
        flags.zero_()
        chk, missing = structure()
        if int(flags.sum().item()):
            raise RuntimeError("structure check flags a line the host accepted")

    if nnz != 2 * m:
        raise MetisParseError(
            f"line {header_no}: header declares {m} edges but adjacency lists "
            f"hold {nnz} entries (expected {2 * m})")
    if chk & (CHK_ASYM | CHK_PARALLEL):
        u, v = divmod(missing, n) if missing >= 0 else (0, 0)
        raise MetisParseError(
            f"asymmetric adjacency: vertex {u + 1} lists {v + 1} but not vice versa")
    if chk & CHK_EW_ASYM:
        raise MetisParseError("edge weight differs between the two directions of an edge")

    if coord_source is None:
        coords = np.zeros((n, 2), dtype=np.float64)
    else:
        coords = load_coords(coord_source, expect_n=n)
    g = GeometricGraph(_to_host(offsets), _to_host(neighbors), coords,
                       np.ones(n, dtype=np.float64) if vw is None else _to_host(vw),
                       None if ew is None else _to_host(ew))
    g.validate(_checked=chk)
    return g


# ---------------------------------------------------------------- np.loadtxt tables
def _table(source, want_int: bool, what: str):
    """Values of a whitespace table as np.loadtxt reads it (fileio.py:222, :250): a
    device tensor of the row-major values, plus (rows, columns)."""
    import torch

    from . import _native as N

    buf = _read_bytes(source)
    if buf.shape[0] == 0:
        return None, 0, 0
    tk = _tokenize(buf, ord("#"))
    if tk.n_tokens == 0:
        return None, 0, 0
    sh = torch.cuda.current_stream().cuda_stream
    out = torch.empty(tk.n_tokens, dtype=torch.int64 if want_int else torch.float64, device="cuda")
    info = torch.empty(4, dtype=torch.int64, device="cuda")
    N.call("gp_table_values", tk.line_tok0.data_ptr(), tk.n_lines, tk.tok_val.data_ptr(),
           tk.tok_kind.data_ptr(), tk.n_tokens, int(want_int), out.data_ptr(), info.data_ptr(), sh)
    rows, ragged_line, bad_tok, ncols = (int(v) for v in info.cpu().tolist())
    dtype_name = "int64" if want_int else "float64"
    np_dtype = np.int64 if want_int else np.float64

    def data_row(line: int) -> int:  # 0-based index of `line` among the non-blank lines
        lt = tk.line_tok0
        return int((lt[1:line + 1] > lt[:line]).sum().item())

    bad_line, bad_msg = None, None
    if bad_tok >= 0:
        # numpy's own converter decides every token outside the plain decimal grammar
        kinds = tk.tok_kind[:tk.n_tokens]
        import warnings

        odd = torch.nonzero(kinds != TOK_INT if want_int else kinds > TOK_REAL).flatten()
        lines = (torch.searchsorted(tk.line_tok0, odd, right=True) - 1)
        col0 = (odd - tk.line_tok0[lines]).cpu().tolist()
        lines = lines.cpu().tolist()
        texts = {l: t.split("#", 1)[0].split() for l, t in tk.lines_text(lines).items()}
        fixed_t, fixed_v = [], []
        for t, line, c in zip(odd.cpu().tolist(), lines, col0):
            tok = texts[line][c]
            try:
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    val = np.loadtxt(io.StringIO(tok), dtype=np_dtype, ndmin=1, comments=None)
                fixed_t.append(t)
                fixed_v.append(val[0].item())
            except ValueError:
                bad_line = line
                bad_msg = (f"could not convert string {tok!r} to {dtype_name} at row "
                           f"{data_row(line)}, column {c + 1}.")
                break
        if fixed_t:
            out[torch.tensor(fixed_t, dtype=torch.int64, device="cuda")] = \
                torch.tensor(fixed_v, dtype=out.dtype, device="cuda")
    if ragged_line >= 0 and (bad_line is None or ragged_line <= bad_line):
        nt = int((tk.line_tok0[ragged_line + 1] - tk.line_tok0[ragged_line]).item())
        bad_msg = (f"the number of columns changed from {ncols} to {nt} at row "
                   f"{data_row(ragged_line) + 1}; use `usecols` to select a subset and avoid "
                   "this error")
    if bad_msg is not None:
        raise MetisParseError(f"malformed {what} file: {bad_msg}")
    return out, rows, ncols


def load_coords(source, expect_n: int | None = None) -> np.ndarray:
    """Read a coordinate file: one line per vertex, 2 or 3 reals each (fileio.py:219-237)."""
    import torch

    vals, rows, ncols = _table(source, False, "coordinate")
    if vals is None:
        raise MetisParseError("empty coordinate file")
    if ncols not in (2, 3):
        raise MetisParseError(f"coordinates must have 2 or 3 columns, got {ncols}")
    if expect_n is not None and rows != expect_n:
        raise MetisParseError(f"coordinate file has {rows} lines, expected {expect_n}")
    if not bool(torch.isfinite(vals).all().item()):
        raise MetisParseError("non-finite coordinate")
    from . import staging

    coords = np.empty((rows, ncols), dtype=np.float64)
    staging.d2h_into(coords, vals)
    return coords


def read_partition(source, expect_n: int | None = None, k: int | None = None) -> Partition:
    """Read a partition file: one block id per line (fileio.py:246-263)."""
    vals, rows, ncols = _table(source, True, "partition")
    if vals is None:
        a = np.empty(0, dtype=np.int64)
    else:
        if rows > 1 and ncols > 1:
            raise MetisParseError("partition file must hold one block id per line")
        a = _to_host(vals)
    if expect_n is not None and a.shape[0] != expect_n:
        raise MetisParseError(f"partition file has {a.shape[0]} lines, expected {expect_n}")
    if a.size and int(vals.min().item()) < 0:
        raise MetisParseError("negative block id")
    if k is None:
        k = int(vals.max().item()) + 1 if a.size else 1
    return Partition(assignment=a, k=k)


def write_partition(partition, sink) -> None:
    """Write a partition as one decimal block id per line (fileio.py:271-278), formatted
    on the device (gp_format_ints)."""
    import torch

    from . import _native as N

    a = partition.assignment if hasattr(partition, "assignment") else np.asarray(partition)
    if isinstance(a, np.ndarray):
        if a.dtype.kind == "f":  # the reference writes str(int(x))
            a = np.trunc(a)
        a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).cuda()
    a = a.to(device="cuda", dtype=torch.int64).contiguous().flatten()
    n = int(a.shape[0])
    if n == 0:
        _write_bytes(sink, b"\n")
        return
    sh = torch.cuda.current_stream().cuda_stream
    wsb = N.size_query("gp_format_ints_workspace_bytes", n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    total = torch.empty(1, dtype=torch.int64, device="cuda")
    N.call("gp_format_ints_plan", a.data_ptr(), n, total.data_ptr(), ws.data_ptr(), wsb, sh)
    nbytes = int(total.item())
    out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    N.call("gp_format_ints_write", a.data_ptr(), n, out.data_ptr(), ws.data_ptr(), sh)
    from . import staging

    host = np.empty(nbytes, dtype=np.uint8)
    staging.d2h_into(host, out)
    _write_bytes(sink, host.tobytes() if not isinstance(sink, (str, Path)) else host)


# ---------------------------------------------------------------- generator-side writers
def _num_token(x: float) -> str:
    return str(int(x)) if float(x).is_integer() else repr(float(x))


def write_metis_graph(graph: GeometricGraph, sink) -> None:
    """Write the adjacency part of a graph in METIS format (fileio.py:199-216); host
    side (the generator's output, not on the partition path)."""
    has_vwgt = not np.all(graph.vertex_weights == 1.0)
    has_ewgt = graph.edge_weights is not None
    head = f"{graph.n} {graph.m}"
    if has_vwgt or has_ewgt:
        head += f" 0{int(has_vwgt)}{int(has_ewgt)}"
    rows = [head]
    nbr1 = (graph.neighbors + 1).tolist()
    ews = [_num_token(x) for x in graph.edge_weights] if has_ewgt else None
    off = graph.offsets.tolist()
    for u in range(graph.n):
        toks = [_num_token(graph.vertex_weights[u])] if has_vwgt else []
        for j in range(off[u], off[u + 1]):
            toks.append(str(nbr1[j]))
            if has_ewgt:
                toks.append(ews[j])
        rows.append(" ".join(toks))
    _write_bytes(sink, ("\n".join(rows) + "\n").encode("ascii"))


def write_coords(coords: np.ndarray, sink) -> None:
    """Write coordinates, one vertex per line, full float64 precision (fileio.py:240-243)."""
    s = io.StringIO()
    np.savetxt(s, np.asarray(coords, dtype=np.float64), fmt="%.17g")
    _write_bytes(sink, s.getvalue().encode("ascii"))
