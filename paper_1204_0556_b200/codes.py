"""Parity-check matrices, the Tanner-graph edge layout, alist I/O and code
construction.

Host-side mirror of the reference's ``polylp.codes`` module
(``/root/reference/pkg/src/polylp/codes.py``).  ``ParityCheckMatrix`` keeps
the reference's public surface -- ``n_vars``, ``n_checks``,
``check_neighborhoods``, ``var_neighborhoods``, ``edge_var``, ``check_ptr``,
``checks_by_degree``, ``var_degrees``, ``n_edges``, ``from_dense``,
``to_dense``, ``design_rate``, equality and plain-data pickling
(codes.py:24-142) -- so a caller can hand the same object to the reference
and to this package.  Edge order is the reference's: edges grouped by check,
checks in index order, variables sorted inside a check (codes.py:42, 91-99).

What is new here:

* ``gen_regular_ldpc`` keeps the reference's rejection sampler and its
  exact draw sequence (codes.py:263-287), so it returns the reference's
  matrix for every seed where the reference succeeds.
* ``make_ldpc`` is the builder's own generator for the benchmark codes: a
  configuration-model draw whose parallel edges are *repaired* by socket
  swaps instead of redrawing the whole permutation, followed (optionally) by
  4-cycle removal to girth >= 6.  The reference sampler cannot build the
  (3,13) n=1040 code at all.
"""

from __future__ import annotations

import functools

from functools import cached_property

import numpy as np
from numpy.typing import ArrayLike, NDArray


class AlistParseError(ValueError):
    """Malformed alist text; the message names the offending line (codes.py:16)."""


class CodeGenerationError(RuntimeError):
    """Random ensemble sampling failed within the retry budget (codes.py:20)."""


class ParityCheckMatrix:
    """Sparse M x N parity-check matrix (mirror of codes.py:24-142).

    ``check_neighborhoods[j]`` is the sorted variable list of check ``j``.
    Instances are immutable and safe to share; the device-resident copy of
    the graph is built lazily by :mod:`paper_1204_0556_b200.admm_decoder`
    and cached per device on the instance.
    """

    def __init__(self, n_vars: int, check_neighborhoods: list[ArrayLike]):
        if n_vars <= 0:
            raise ValueError("n_vars must be positive")
        if not check_neighborhoods:
            raise ValueError("need at least one check")
        rows: list[NDArray[np.int64]] = []
        for j, nb in enumerate(check_neighborhoods):
            row = np.sort(np.asarray(nb, dtype=np.int64).reshape(-1))
            if row.size == 0:
                raise ValueError(f"check {j} has no variables")
            if row[0] < 0 or row[-1] >= n_vars:
                raise ValueError(f"check {j} has a variable index out of range")
            if row.size > 1 and np.any(row[1:] == row[:-1]):
                raise ValueError(f"check {j} has a parallel edge")
            row.flags.writeable = False
            rows.append(row)
        self.n_vars = int(n_vars)
        self.n_checks = len(rows)
        self.check_neighborhoods: tuple[NDArray[np.int64], ...] = tuple(rows)
        self._device_graphs: dict = {}

    # -- construction helpers ------------------------------------------------
    @classmethod
    def from_dense(cls, h: ArrayLike) -> "ParityCheckMatrix":
        h = np.asarray(h)
        if h.ndim != 2:
            raise ValueError("dense parity-check matrix must be 2-D")
        return cls(h.shape[1], [np.nonzero(row)[0] for row in h])

    def to_dense(self) -> NDArray[np.uint8]:
        h = np.zeros((self.n_checks, self.n_vars), dtype=np.uint8)
        h[np.repeat(np.arange(self.n_checks), self.check_degrees), self.edge_var] = 1
        return h

    # -- Tanner-graph views (codes.py:79-115) --------------------------------
    @cached_property
    def check_degrees(self) -> NDArray[np.int64]:
        return np.fromiter((r.size for r in self.check_neighborhoods), np.int64, self.n_checks)

    @cached_property
    def edge_var(self) -> NDArray[np.int64]:
        """Variable of every edge, edges grouped by check (codes.py:91-94)."""
        ev = np.concatenate(self.check_neighborhoods).astype(np.int64)
        ev.flags.writeable = False
        return ev

    @cached_property
    def edge_check(self) -> NDArray[np.int64]:
        ec = np.repeat(np.arange(self.n_checks, dtype=np.int64), self.check_degrees)
        ec.flags.writeable = False
        return ec

    @cached_property
    def check_ptr(self) -> NDArray[np.int64]:
        """CSR offsets: edges of check j are check_ptr[j]:check_ptr[j+1] (codes.py:96-99)."""
        ptr = np.zeros(self.n_checks + 1, dtype=np.int64)
        np.cumsum(self.check_degrees, out=ptr[1:])
        ptr.flags.writeable = False
        return ptr

    @cached_property
    def var_degrees(self) -> NDArray[np.int64]:
        return np.bincount(self.edge_var, minlength=self.n_vars).astype(np.int64)

    @cached_property
    def var_edges(self) -> tuple[NDArray[np.int64], NDArray[np.int64]]:
        """CSC edge map: (var_ptr[N+1], edge ids grouped by variable).

        Edges of variable i are listed in increasing edge id, i.e. in
        increasing check index -- the order in which the reference's
        ``np.bincount`` accumulates them (admm_decoder.py:116).
        """
        order = np.argsort(self.edge_var, kind="stable")
        ptr = np.zeros(self.n_vars + 1, dtype=np.int64)
        np.cumsum(self.var_degrees, out=ptr[1:])
        return ptr, order.astype(np.int64)

    @cached_property
    def var_neighborhoods(self) -> tuple[NDArray[np.int64], ...]:
        ptr, eids = self.var_edges
        checks = self.edge_check[eids]
        out = []
        for i in range(self.n_vars):
            a = np.array(checks[ptr[i]:ptr[i + 1]], dtype=np.int64)
            a.flags.writeable = False
            out.append(a)
        return tuple(out)

    @property
    def n_edges(self) -> int:
        return int(self.check_ptr[-1])

    def check_slice(self, j: int) -> slice:
        return slice(int(self.check_ptr[j]), int(self.check_ptr[j + 1]))

    @cached_property
    def checks_by_degree(self) -> dict[int, NDArray[np.int64]]:
        """Edge-index matrix (m_d, d) per distinct check degree (codes.py:104-115)."""
        out: dict[int, NDArray[np.int64]] = {}
        for d in np.unique(self.check_degrees):
            js = np.nonzero(self.check_degrees == d)[0]
            rows = self.check_ptr[js][:, None] + np.arange(int(d))[None, :]
            rows.flags.writeable = False
            out[int(d)] = rows
        return out

    @property
    def design_rate(self) -> float:
        return 1.0 - self.n_checks / self.n_vars

    @property
    def max_check_degree(self) -> int:
        return int(self.check_degrees.max())

    @property
    def max_var_degree(self) -> int:
        return int(self.var_degrees.max()) if self.n_vars else 0

    def girth_at_least_6(self) -> bool:
        """True when no two checks share two or more variables (no 4-cycles)."""
        h = self.to_dense().astype(np.int32)
        ov = h @ h.T
        np.fill_diagonal(ov, 0)
        return bool(ov.max(initial=0) < 2)

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, ParityCheckMatrix):
            return NotImplemented
        return (
            self.n_vars == other.n_vars
            and self.n_checks == other.n_checks
            and all(np.array_equal(a, b) for a, b in zip(self.check_neighborhoods, other.check_neighborhoods))
        )

    def __hash__(self) -> int:  # identity hash: instances are immutable value objects
        return id(self)

    def __repr__(self) -> str:
        return f"ParityCheckMatrix(n_vars={self.n_vars}, n_checks={self.n_checks})"

    def __getstate__(self) -> dict:
        return {"n_vars": self.n_vars, "checks": [np.asarray(a) for a in self.check_neighborhoods]}

    def __setstate__(self, state: dict) -> None:
        self.__init__(state["n_vars"], state["checks"])

    @classmethod
    def from_reference(cls, code) -> "ParityCheckMatrix":
        """Adopt any object exposing ``n_vars`` and ``check_neighborhoods``
        (for example a reference ``polylp.ParityCheckMatrix``)."""
        return cls(int(code.n_vars), [np.asarray(a) for a in code.check_neighborhoods])


def as_code(code) -> ParityCheckMatrix:
    """Accept this package's matrix or any duck-typed reference matrix."""
    if isinstance(code, ParityCheckMatrix):
        return code
    if hasattr(code, "n_vars") and hasattr(code, "check_neighborhoods"):
        cached = getattr(code, "_b200_mirror", None)
        if cached is None:
            cached = ParityCheckMatrix.from_reference(code)
            try:
                object.__setattr__(code, "_b200_mirror", cached)
            except (AttributeError, TypeError):
                pass
        return cached
    raise TypeError("expected a ParityCheckMatrix")


def is_codeword(code, x: ArrayLike) -> bool:
    """True iff every check of ``x`` has even parity (codes.py:145-154)."""
    code = as_code(code)
    x = np.asarray(x)
    if x.shape != (code.n_vars,):
        raise ValueError(f"expected a length-{code.n_vars} vector")
    if not np.all((x == 0) | (x == 1)):
        raise ValueError("codeword entries must be 0 or 1")
    bits = x.astype(np.int64)[code.edge_var]
    parity = np.zeros(code.n_checks, dtype=np.int64)
    np.add.at(parity, code.edge_check, bits)
    return not bool(np.any(parity & 1))


# --------------------------------------------------------------------------
# alist text format (codes.py:157-260)
# --------------------------------------------------------------------------
def _ints(lines: list[str], idx: int, what: str) -> list[int]:
    if idx >= len(lines):
        raise AlistParseError(f"line {idx + 1}: missing {what}")
    try:
        return [int(t) for t in lines[idx].split()]
    except ValueError as exc:
        raise AlistParseError(f"line {idx + 1}: non-integer token in {what}") from exc


def parse_alist(text: str) -> ParityCheckMatrix:
    """Parse alist text (N M / max degrees / column degrees / row degrees /
    N column lines / M row lines; 1-based, zero padding ignored)."""
    lines = text.splitlines()
    while lines and not lines[-1].strip():
        lines.pop()
    head = _ints(lines, 0, "size header")
    if len(head) != 2:
        raise AlistParseError("line 1: expected 'N M'")
    n, m = head
    if n <= 0 or m <= 0:
        raise AlistParseError("line 1: dimensions must be positive")
    maxd = _ints(lines, 1, "maximum degrees")
    if len(maxd) != 2:
        raise AlistParseError("line 2: expected maximum column and row degree")
    col_deg = _ints(lines, 2, "column degrees")
    if len(col_deg) != n:
        raise AlistParseError(f"line 3: expected {n} column degrees, got {len(col_deg)}")
    row_deg = _ints(lines, 3, "row degrees")
    if len(row_deg) != m:
        raise AlistParseError(f"line 4: expected {m} row degrees, got {len(row_deg)}")
    if any(d < 0 or d > maxd[0] for d in col_deg):
        raise AlistParseError("line 3: column degree exceeds declared maximum")
    if any(d < 1 or d > maxd[1] for d in row_deg):
        raise AlistParseError("line 4: row degree out of range")
    want = 4 + n + m
    if len(lines) != want:
        raise AlistParseError(f"line {min(len(lines), want) + 1}: expected {want} lines, got {len(lines)}")
    cols = []
    for k in range(n):
        ent = [e for e in _ints(lines, 4 + k, "column entries") if e != 0]
        if len(ent) != col_deg[k]:
            raise AlistParseError(
                f"line {5 + k}: column {k + 1} lists {len(ent)} checks, degree says {col_deg[k]}")
        if any(e < 1 or e > m for e in ent):
            raise AlistParseError(f"line {5 + k}: check index out of range")
        cols.append(sorted(e - 1 for e in ent))
    rows = []
    for k in range(m):
        ln = 4 + n + k
        ent = [e for e in _ints(lines, ln, "row entries") if e != 0]
        if len(ent) != row_deg[k]:
            raise AlistParseError(
                f"line {ln + 1}: row {k + 1} lists {len(ent)} variables, degree says {row_deg[k]}")
        if any(e < 1 or e > n for e in ent):
            raise AlistParseError(f"line {ln + 1}: variable index out of range")
        rows.append(sorted(e - 1 for e in ent))
    seen: list[set[int]] = [set() for _ in range(m)]
    for i, cs in enumerate(cols):
        for j in cs:
            seen[j].add(i)
    for j in range(m):
        if seen[j] != set(rows[j]):
            raise AlistParseError(f"line {4 + n + j + 1}: row {j + 1} disagrees with the column section")
    return ParityCheckMatrix(n, rows)


def emit_alist(code: ParityCheckMatrix) -> str:
    """Canonical alist text: unpadded, single-spaced, 1-based (codes.py:248-260)."""
    code = as_code(code)
    out = [
        f"{code.n_vars} {code.n_checks}",
        f"{code.max_var_degree} {code.max_check_degree}",
        " ".join(str(int(d)) for d in code.var_degrees),
        " ".join(str(int(d)) for d in code.check_degrees),
    ]
    out += [" ".join(str(int(c) + 1) for c in nb) for nb in code.var_neighborhoods]
    out += [" ".join(str(int(v) + 1) for v in nb) for nb in code.check_neighborhoods]
    return "\n".join(out) + "\n"


# --------------------------------------------------------------------------
# Code construction
# --------------------------------------------------------------------------
def _check_params(n: int, dv: int, dc: int) -> int:
    if n <= 0 or dv <= 0 or dc <= 0:
        raise ValueError("code parameters must be positive")
    if (n * dv) % dc:
        raise ValueError("n * var_deg must be divisible by check_deg")
    return n * dv // dc


def gen_regular_ldpc(n: int, var_deg: int, check_deg: int, seed: int,
                     max_attempts: int = 1000) -> ParityCheckMatrix:
    """Reference-compatible rejection sampler (codes.py:263-287).

    Same RNG stream as the reference (``default_rng(seed)`` then one
    ``permutation`` of the socket list per attempt), so the matrices agree
    wherever the reference succeeds; raises ``CodeGenerationError`` where it
    would.
    """
    m = _check_params(n, var_deg, check_deg)
    rng = np.random.default_rng(seed)
    sockets = np.repeat(np.arange(n), var_deg)
    for _ in range(max_attempts):
        deal = np.sort(rng.permutation(sockets).reshape(m, check_deg), axis=1)
        if not np.any(deal[:, 1:] == deal[:, :-1]):
            return ParityCheckMatrix(n, list(deal))
    raise CodeGenerationError(
        f"no parallel-edge-free ({var_deg},{check_deg}) code of length {n} found in {max_attempts} attempts")


class _Deal:
    """Mutable socket deal: ``rows[j]`` is the variable list of check j."""

    def __init__(self, rows: np.ndarray, n: int):
        self.rows = rows  # (m, dc) int64
        self.n = n
        self.m = rows.shape[0]
        self.var_checks: list[list[int]] = [[] for _ in range(n)]
        for j in range(self.m):
            for v in rows[j]:
                self.var_checks[int(v)].append(j)

    def has_parallel(self, j: int) -> bool:
        r = self.rows[j]
        return len(set(r.tolist())) != r.size

    def score(self, j: int, girth6: bool) -> int:
        """Defects of check j: duplicated sockets plus (with ``girth6``) the
        number of other checks sharing two or more variables with it."""
        row = self.rows[j].tolist()
        uniq = set(row)
        bad = len(row) - len(uniq)
        if girth6:
            count: dict[int, int] = {}
            for v in uniq:
                for c in self.var_checks[v]:
                    if c != j:
                        count[c] = count.get(c, 0) + 1
            bad += sum(1 for k in count.values() if k >= 2)
        return bad

    def offending_slots(self, j: int) -> list[int]:
        row = self.rows[j].tolist()
        seen: dict[int, int] = {}
        out = []
        for s, v in enumerate(row):
            if v in seen:
                out.append(s)
            seen[v] = s
        if out:
            return out
        count: dict[int, int] = {}
        for v in set(row):
            for c in self.var_checks[v]:
                if c != j:
                    count[c] = count.get(c, 0) + 1
        partners = {c for c, k in count.items() if k >= 2}
        return [s for s, v in enumerate(row) if any(c in partners for c in self.var_checks[v] if c != j)]

    def swap(self, j1: int, s1: int, j2: int, s2: int) -> None:
        a, b = int(self.rows[j1, s1]), int(self.rows[j2, s2])
        self.var_checks[a].remove(j1)
        self.var_checks[b].remove(j2)
        self.rows[j1, s1], self.rows[j2, s2] = b, a
        self.var_checks[b].append(j1)
        self.var_checks[a].append(j2)


def make_ldpc(n: int, var_deg: int, check_deg: int, seed: int = 0, *,
              girth6: bool = True, max_swaps: int | None = None) -> ParityCheckMatrix:
    """Random (var_deg, check_deg)-regular code with repaired parallel edges.

    1. Configuration model: ``default_rng(seed).permutation`` of the socket
       list dealt to checks (the same first draw as the reference sampler).
    2. Every parallel edge is repaired by swapping one of its sockets with a
       random socket of another check, accepted only when neither check ends
       up with a parallel edge.
    3. With ``girth6`` every pair of checks sharing two variables (a 4-cycle)
       is broken by the same kind of swap, accepted only when both touched
       checks are free of parallel edges and 4-cycles afterwards.

    Degrees are preserved exactly.  Deterministic per seed.
    """
    m = _check_params(n, var_deg, check_deg)
    rng = np.random.default_rng(seed)
    sockets = np.repeat(np.arange(n), var_deg)
    deal = _Deal(rng.permutation(sockets).reshape(m, check_deg).astype(np.int64), n)
    budget = max_swaps if max_swaps is not None else 200 * m * check_deg

    def fail() -> CodeGenerationError:
        return CodeGenerationError(
            f"could not repair ({var_deg},{check_deg}) code of length {n} (seed {seed})")

    # A swap is accepted when it lowers the joint defect count of the two
    # checks it touches (or, with probability 0.3, leaves it unchanged, which
    # lets the search leave plateaus); sweeps repeat until every check is clean.
    dirty = [j for j in range(m) if deal.score(j, girth6)]
    while dirty:
        for j in dirty:
            cur = deal.score(j, girth6)
            tries = 0
            while cur and tries < 4000:
                slots = deal.offending_slots(j)
                s1 = slots[int(rng.integers(len(slots)))]
                j2 = int(rng.integers(m))
                if j2 == j:
                    continue
                s2 = int(rng.integers(check_deg))
                tries += 1
                budget -= 1
                if budget < 0:
                    raise fail()
                before = cur + deal.score(j2, girth6)
                deal.swap(j, s1, j2, s2)
                new = deal.score(j, girth6)
                after = new + deal.score(j2, girth6)
                if after < before or (after == before and rng.random() < 0.3):
                    cur = new
                else:
                    deal.swap(j, s1, j2, s2)
        dirty = [j for j in range(m) if deal.score(j, girth6)]
    rows = [np.sort(deal.rows[j]) for j in range(m)]
    return ParityCheckMatrix(n, rows)


#: The BASELINE.json benchmark codes: name -> (n, var_deg, check_deg, girth6).
BASELINE_CODES = {
    "cfg1_n96": (96, 3, 6, False),
    "cfg2_n1008": (1008, 3, 6, True),
    "cfg3_n2640": (2640, 3, 6, True),
    "cfg4_n1040": (1040, 3, 13, True),
    "cfg5_n16384": (16384, 3, 6, True),
}


@functools.lru_cache(maxsize=None)
def baseline_code(name: str, seed: int = 0) -> ParityCheckMatrix:
    """The BASELINE code `name` (cached: a ParityCheckMatrix is immutable, and
    its device graphs are cached on it)."""
    n, dv, dc, g6 = BASELINE_CODES[name]
    return make_ldpc(n, dv, dc, seed, girth6=g6)
