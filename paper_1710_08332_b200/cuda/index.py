"""Index arithmetic for generated kernels.

Every array subscript the emitter produces (loop variables, literals, and the
`*`, `+`, `/`, `%` introduced by split/join/transpose/asVector access paths)
is kept as a canonical polynomial over *atoms*: loop or size variables and
irreducible floor-divisions / remainders.  Division and remainder by a
constant are cancelled whenever the loop ranges prove the remainder term lies
in [0, n) -- the contract of the reference's `_IndexSimplifier`
(SRC/codegen_c.py:78-193) -- so `(i*8 + j) / 8` renders as `i` and
`(i*8 + j) % 8` as `j` when `j < 8`.  Additionally nested divisions fold
(`(x/a)/b == x/(a*b)`), and a maximum-value analysis decides per subscript
whether 32-bit arithmetic is safe or 64-bit is required (the reference uses
`int` everywhere, which overflows at N = 2^31, SURVEY.md finding 3).
"""
from __future__ import annotations

from typing import Dict, Mapping, Optional, Tuple

INT32_MAX = 2 ** 31 - 1

# atom key -> ("v", name) | ("d", Ix, n) | ("m", Ix, n) | ("x", Ix, Ix)  (xor)
_ATOMS: Dict[str, tuple] = {}


def _atom(key: str, node: tuple) -> str:
    _ATOMS.setdefault(key, node)
    return key


class Ix:
    __slots__ = ("terms",)

    def __init__(self, terms=()):
        acc: Dict[Tuple[str, ...], int] = {}
        for mono, c in terms:
            if c:
                k = tuple(sorted(mono))
                acc[k] = acc.get(k, 0) + c
        self.terms = tuple(sorted(((m, c) for m, c in acc.items() if c),
                                  key=lambda mc: (len(mc[0]), mc[0])))

    # ---------------------------------------------------------- algebra
    def __add__(self, o: "IxLike") -> "Ix":
        return Ix(self.terms + ix(o).terms)

    __radd__ = __add__

    def __mul__(self, o: "IxLike") -> "Ix":
        o = ix(o)
        return Ix((m1 + m2, c1 * c2) for m1, c1 in self.terms for m2, c2 in o.terms)

    __rmul__ = __mul__

    def __eq__(self, o) -> bool:
        return isinstance(o, Ix) and self.terms == o.terms

    def __hash__(self):
        return hash(self.terms)

    def __repr__(self):
        return f"Ix({render(self)})"

    @property
    def const(self) -> Optional[int]:
        if not self.terms:
            return 0
        if len(self.terms) == 1 and self.terms[0][0] == ():
            return self.terms[0][1]
        return None

    def var_name(self) -> Optional[str]:
        """Name if this index is exactly one variable."""
        if len(self.terms) == 1 and self.terms[0][1] == 1 and len(self.terms[0][0]) == 1:
            node = _ATOMS[self.terms[0][0][0]]
            if node[0] == "v":
                return node[1]
        return None

    def atoms(self):
        for mono, _ in self.terms:
            for a in mono:
                yield a


IxLike = "Ix | int | str"


def ix(x) -> Ix:
    if isinstance(x, Ix):
        return x
    if isinstance(x, int):
        return Ix([((), x)])
    if isinstance(x, str):
        return Ix([((_atom(x, ("v", x)),), 1)])
    raise TypeError(f"not an index: {x!r}")


def var(name: str) -> Ix:
    return ix(name)


# ----------------------------------------------------------- ranges

def max_value(e: Ix, R: Mapping[str, Optional[int]]) -> Optional[int]:
    """Largest value e can take (all atoms are >= 0); None if unbounded."""
    total = 0
    for mono, c in e.terms:
        if c < 0:
            return None
        t = c
        for a in mono:
            m = _atom_max(a, R)
            if m is None:
                return None
            t *= m
        total += t
    return total


def _atom_max(key: str, R) -> Optional[int]:
    node = _ATOMS[key]
    if node[0] == "v":
        b = R.get(node[1])
        return None if b is None else b - 1
    if node[0] == "x":
        ma, mb = max_value(node[1], R), max_value(node[2], R)
        if ma is None or mb is None:
            return None
        return (1 << max(ma, mb).bit_length()) - 1
    inner = max_value(node[1], R)
    if node[0] == "d":
        return None if inner is None else inner // node[2]
    return node[2] - 1 if inner is None else min(inner, node[2] - 1)


def _split_multiples(e: Ix, n: int):
    q = Ix((m, c // n) for m, c in e.terms if c % n == 0)
    r = Ix((m, c) for m, c in e.terms if c % n != 0)
    return q, r


def _common_factor(r: Ix, n: int, R) -> int:
    """Largest proper divisor g of n with r = g*X + s, 0 <= s < g provable.
    Then floor(r/n) = floor(X/(n/g)) and r % n = g*(X % (n/g)) + s."""
    from math import gcd
    cands = {gcd(n, c) for _, c in r.terms} | {1 << k for k in range(1, 40) if n % (1 << k) == 0}
    for g in sorted(cands, reverse=True):
        if g <= 1 or g >= n or n % g:
            continue
        big, small = _split_multiples(r, g)
        if not big.terms:
            continue
        ms = max_value(small, R)
        if ms is not None and ms < g:
            return g
    return 0


def div(e, n: int, R) -> Ix:
    """floor(e / n) for e >= 0, n > 0."""
    e = ix(e)
    if n == 1:
        return e
    # (x / a) / n == x / (a*n)
    if len(e.terms) == 1 and e.terms[0][1] == 1 and len(e.terms[0][0]) == 1:
        node = _ATOMS[e.terms[0][0][0]]
        if node[0] == "d":
            return div(node[1], node[2] * n, R)
    q, r = _split_multiples(e, n)
    if not r.terms:
        return q
    mr = max_value(r, R)
    if mr is not None and mr < n:
        return q
    if mr is not None and r.const is not None:
        return q + (r.const // n)
    g = _common_factor(r, n, R)
    if g:
        big, small = _split_multiples(r, g)
        return q + div(big, n // g, R)
    key = f"({render(r)})/{n}"
    return q + Ix([((_atom(key, ("d", r, n)),), 1)])


def mod(e, n: int, R) -> Ix:
    """e % n for e >= 0, n > 0."""
    e = ix(e)
    if n == 1:
        return Ix()
    _q, r = _split_multiples(e, n)
    if not r.terms:
        return Ix()
    mr = max_value(r, R)
    if mr is not None and mr < n:
        return r
    if r.const is not None:
        return ix(r.const % n)
    g = _common_factor(r, n, R)
    if g:
        big, small = _split_multiples(r, g)
        return mod(big, n // g, R) * g + small
    key = f"({render(r)})%{n}"
    return Ix([((_atom(key, ("m", r, n)),), 1)])


def xor(a, b) -> Ix:
    """a ^ b as an opaque atom (shared-memory swizzles); both non-negative."""
    a, b = ix(a), ix(b)
    if not b.terms:
        return a
    key = f"({render(a)})^({render(b)})"
    return Ix([((_atom(key, ("x", a, b)),), 1)])


# ---------------------------------------------------------- rendering

def render(e: Ix, R: Optional[Mapping[str, Optional[int]]] = None, wide: Optional[bool] = None) -> str:
    """C text.  wide=None decides from the range analysis (R given) whether a
    64-bit evaluation is needed; True forces `(long long)` promotion."""
    if wide is None:
        wide = R is not None and (max_value(e, R) is None or max_value(e, R) > INT32_MAX)
    if not e.terms:
        return "0"
    parts = []
    for mono, c in sorted(e.terms, key=lambda mc: (-len(mc[0]), mc[0])):
        factors = [_render_atom(a, R, wide) for a in mono]
        if c != 1 or not factors:
            factors.insert(0, str(c) + ("LL" if wide and not mono else ""))
        if wide and mono:
            factors[0] = f"(long long){factors[0]}"
        parts.append(" * ".join(factors))
    return " + ".join(parts)


def _render_atom(key: str, R, wide: bool) -> str:
    node = _ATOMS[key]
    if node[0] == "v":
        return node[1]
    if node[0] == "x":
        return f"(({render(node[1], R, wide)}) ^ ({render(node[2], R, wide)}))"
    inner_wide = wide or (R is not None and (max_value(node[1], R) is None
                                             or max_value(node[1], R) > INT32_MAX))
    op = "/" if node[0] == "d" else "%"
    return f"(({render(node[1], R, inner_wide)}) {op} {node[2]})"


def evaluate(e: Ix, env: Mapping[str, int]) -> int:
    total = 0
    for mono, c in e.terms:
        t = c
        for a in mono:
            node = _ATOMS[a]
            if node[0] == "v":
                t *= env[node[1]]
            elif node[0] == "d":
                t *= evaluate(node[1], env) // node[2]
            elif node[0] == "x":
                t *= evaluate(node[1], env) ^ evaluate(node[2], env)
            else:
                t *= evaluate(node[1], env) % node[2]
        total += t
    return total


def free_names(e: Ix) -> set:
    out = set()
    for a in e.atoms():
        node = _ATOMS[a]
        if node[0] == "v":
            out.add(node[1])
        elif node[0] == "x":
            out |= free_names(node[1]) | free_names(node[2])
        else:
            out |= free_names(node[1])
    return out
