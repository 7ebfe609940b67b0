"""S-expression surface syntax: tokens, forms, types, and whole programs.

Accepts the reference's `.dpia` language unchanged (`SRC/parser.py:57-259`):
``(nat n)`` / ``(param x TYPE)`` declarations followed by one body phrase,
``;;`` comments, sizes written as ``(* n 1024)``.  Elaboration of the body
(local inference of size and type arguments) lives in `elab.py`.
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple, Union

from .dtypes import (COMM, NUM, AccT, Array, DataType, DepFnT, ExpT, FnT, Idx,
                     Pair, PhraseType, ProdT, VECTOR_WIDTHS, Vector, is_passive,
                     var_t)
from .sizes import Nat, nat


class ParseError(Exception):
    """Unreadable input (CLI exit code 2)."""

    def __init__(self, message: str, line: int = 0, col: int = 0):
        super().__init__(f"{line}:{col}: {message}" if line else message)
        self.message, self.line, self.col = message, line, col


class ElabError(ParseError):
    """Readable input that does not elaborate to a well-typed phrase
    (reported as a type error, CLI exit code 3)."""


@dataclass(frozen=True)
class Token:
    text: str
    line: int
    col: int


SExp = Union[Token, list]

# one alternation, tried in order at every position: layout, a `;;` line
# comment, a parenthesis, or an atom (anything up to the next delimiter)
_LEXEME = re.compile(r"(?P<nl>\n)|(?P<ws>[ \t\r]+)|(?P<comment>;;[^\n]*)|(?P<paren>[()])"
                     r"|(?P<atom>[^ \t\r\n();]+)")


def tokenize(text: str) -> List[Token]:
    """Atoms and parentheses with 1-based line / column positions."""
    out: List[Token] = []
    line, line_start, pos = 1, 0, 0
    while pos < len(text):
        m = _LEXEME.match(text, pos)
        if m is None:      # a lone ';' -- the only character no lexeme accepts
            raise ParseError(f"unexpected character {text[pos]!r}", line, pos - line_start + 1)
        kind = m.lastgroup
        if kind == "nl":
            line, line_start = line + 1, m.end()
        elif kind in ("paren", "atom"):
            out.append(Token(m.group(), line, pos - line_start + 1))
        pos = m.end()
    return out


def read_all(text: str) -> List[SExp]:
    """The top-level forms: nested lists of tokens."""
    toks = tokenize(text)

    def form(k: int):
        """The form starting at toks[k] and the index after it."""
        if toks[k].text != "(":
            return toks[k], k + 1
        opener, items, k = toks[k], [], k + 1
        while k < len(toks) and toks[k].text != ")":
            item, k = form(k)
            items.append(item)
        if k == len(toks):
            raise ParseError(f"input ends inside the form opened at {opener.line}:{opener.col}")
        return items, k + 1

    forms, k = [], 0
    while k < len(toks):
        if toks[k].text == ")":
            raise ParseError("')' closes nothing", toks[k].line, toks[k].col)
        f, k = form(k)
        forms.append(f)
    return forms


def position(sx: SExp) -> Tuple[int, int]:
    """(line, column) of the first token inside sx; (0, 0) for ()."""
    first = sx
    while isinstance(first, list) and first:
        first = first[0]
    return (first.line, first.col) if isinstance(first, Token) else (0, 0)


def error_at(sx: SExp, msg: str, cls=ParseError) -> ParseError:
    return cls(msg, *position(sx))


def head_of(sx: SExp) -> Optional[str]:
    """The operator atom of a form, if it has one."""
    return sx[0].text if isinstance(sx, list) and sx and isinstance(sx[0], Token) else None


_INT = re.compile(r"[+-]?\d+")


def number_of(sx: SExp):
    """The int or float a token spells, else None."""
    if not isinstance(sx, Token):
        return None
    if _INT.fullmatch(sx.text):
        return int(sx.text)
    try:
        return float(sx.text)
    except ValueError:
        return None


# ---------------------------------------------------------------- types

def parse_nat(sx: SExp) -> Nat:
    if isinstance(sx, Token):
        v = number_of(sx)
        if v is None:
            return nat(sx.text)
        if isinstance(v, int) and v >= 0:
            return nat(v)
        raise error_at(sx, f"not a size expression: {sx.text}")
    h = head_of(sx)
    if h in ("+", "*") and len(sx) == 3:
        a, b = parse_nat(sx[1]), parse_nat(sx[2])
        return a + b if h == "+" else a * b
    raise error_at(sx, "malformed size expression")


def parse_data(sx: SExp) -> DataType:
    if isinstance(sx, Token):
        if sx.text == "num":
            return NUM
        raise error_at(sx, f"unknown data type: {sx.text}")
    h, k = head_of(sx), len(sx)
    if h == "idx" and k == 2:
        return Idx(parse_nat(sx[1]))
    if h == "array" and k == 3:
        return Array(parse_nat(sx[1]), parse_data(sx[2]))
    if h == "pair" and k == 3:
        return Pair(parse_data(sx[1]), parse_data(sx[2]))
    if h == "vec" and k == 2:
        w = number_of(sx[1])
        if w not in VECTOR_WIDTHS:
            raise error_at(sx, f"illegal vector width: {sx[1]}")
        return Vector(w)
    raise error_at(sx, "malformed data type")


def parse_phrase_type(sx: SExp) -> PhraseType:
    if isinstance(sx, Token):
        if sx.text == "comm":
            return COMM
        raise error_at(sx, f"unknown phrase type: {sx.text}")
    h, k = head_of(sx), len(sx)
    if h in ("exp", "acc", "var") and k == 2:
        d = parse_data(sx[1])
        return {"exp": ExpT, "acc": AccT, "var": var_t}[h](d)
    if h == "prod" and k == 3:
        return ProdT(parse_phrase_type(sx[1]), parse_phrase_type(sx[2]))
    if h in ("->", "->p") and k >= 3:
        out = parse_phrase_type(sx[-1])
        for a in reversed(sx[1:-1]):
            out = FnT(parse_phrase_type(a), out, passive=(h == "->p"))
        return out
    if h == "forall" and k == 3 and isinstance(sx[1], list) and len(sx[1]) == 2:
        name, kind = sx[1][0].text, sx[1][1].text
        if kind not in ("nat", "data"):
            raise error_at(sx, f"unknown kind: {kind}")
        return DepFnT(name, kind, parse_phrase_type(sx[2]))
    raise error_at(sx, "malformed phrase type")


# --------------------------------------------------------------- programs

@dataclass
class SourceProgram:
    """A parsed program (same shape as the reference's, `SRC/parser.py:201-225`)."""
    nat_params: List[str] = field(default_factory=list)
    params: List[Tuple[str, PhraseType]] = field(default_factory=list)
    body: object = None
    body_type: Optional[PhraseType] = None

    @property
    def pi(self) -> Dict[str, PhraseType]:
        return {n: t for n, t in self.params if is_passive(t)}

    @property
    def gamma(self) -> Dict[str, PhraseType]:
        return {n: t for n, t in self.params if not is_passive(t)}

    @property
    def delta(self) -> Dict[str, str]:
        return {n: "nat" for n in self.nat_params}


def parse(text: str) -> SourceProgram:
    from .elab import Elaborator
    prog = SourceProgram()
    body_sx: Optional[SExp] = None
    for form in read_all(text):
        h = head_of(form)
        if h == "nat":
            if len(form) != 2 or not isinstance(form[1], Token):
                raise error_at(form, "expected (nat NAME)")
            prog.nat_params.append(form[1].text)
        elif h == "param":
            if len(form) != 3 or not isinstance(form[1], Token):
                raise error_at(form, "expected (param NAME TYPE)")
            if any(n == form[1].text for n, _ in prog.params):
                raise error_at(form, f"duplicate parameter: {form[1].text}")
            prog.params.append((form[1].text, parse_phrase_type(form[2])))
        elif body_sx is None:
            body_sx = form
        else:
            raise error_at(form, "more than one body phrase")
    if body_sx is None:
        raise ParseError("program has no body phrase")
    try:
        prog.body, prog.body_type = Elaborator(dict(prog.params)).infer(body_sx)
    except ElabError:
        raise
    except ParseError as e:
        raise ElabError(e.message, e.line, e.col) from None
    return prog


def parse_phrase(text: str, env: Optional[Dict[str, PhraseType]] = None):
    from .elab import Elaborator
    forms = read_all(text)
    if len(forms) != 1:
        raise ParseError(f"expected exactly one phrase, got {len(forms)}")
    return Elaborator(dict(env or {})).infer(forms[0])
