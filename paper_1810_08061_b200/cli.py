"""`skb run`: execute a staged program on the B200 from the command line, with
the reference CLI's feed syntax, output format and exit codes (reference
cli.py:34-40, `stagekit run --mode staged`, :184-200).

    python -m paper_1810_08061_b200 run PROGRAM [--feed NAME=SPEC ...]
        [--entry main] [--backend graph|sexpr] [--precision fast|f64]

PROGRAM is a staged graph in one of the wire formats — `.sexpr` (the
reference's `to_sexpr` / `stagekit graph` text), `.json` (skb's IR JSON) — or an
MSL source file, which is traced with the reference's own front end
(`trace_module`, frozen API; needs the `stagekit` package importable).

Exit codes: 0 success, 1 usage, 3 staging failed (feed syntax, tracing),
4 runtime failed.  Diagnostics go to stderr as
`<file>:<line>:<col>: <phase>: <message>`.  Outputs: print log lines, then one
line per result (reference runtime/values.py format_value).
"""

from __future__ import annotations

import argparse
import sys

from .errors import SkbError

EXIT_USAGE, EXIT_STAGING, EXIT_RUNTIME = 1, 3, 4


class _Fail(Exception):
    def __init__(self, phase, message, span=None):
        super().__init__(message)
        self.phase, self.message, self.span = phase, message, span


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        sys.exit(EXIT_USAGE)


def _report(file_name, f: _Fail) -> int:
    span = f.span
    generated = getattr(span, "is_generated", False)
    line = getattr(span, "start_line", 1) if span is not None and not generated else 1
    col = getattr(span, "start_col", 1) if span is not None and not generated else 1
    print(f"{file_name}:{line}:{col}: {f.phase}: {f.message}", file=sys.stderr)
    return {"staging": EXIT_STAGING, "runtime": EXIT_RUNTIME}.get(f.phase, EXIT_USAGE)


def _load_graph(path, entry, backend, feeds):
    from . import ir, sexpr
    if path.endswith(".json"):
        with open(path) as fh:
            return ir.from_json(fh.read())
    if path.endswith(".sexpr"):
        with open(path) as fh:
            return sexpr.from_sexpr(fh.read())
    # MSL source: the reference's own front end traces it (the frozen conversion API)
    try:
        from stagekit.runtime import ParamSpec, trace_module
        from stagekit.syntax import parse_module
        from stagekit.transforms import PassConfig
    except ImportError:
        raise _Fail("usage", "tracing an MSL file needs the stagekit package (or pass a .sexpr/.json graph)")
    with open(path) as fh:
        module = parse_module(fh.read(), path)
    params = []
    for name, v in feeds.items():
        if hasattr(v, "dtype"):
            params.append(ParamSpec(name, v.dtype, tuple(v.shape)))
        else:
            params.append(ParamSpec(name, "tree"))
    try:
        return trace_module(module, entry, params, PassConfig(backend=backend)).graph
    except Exception as exc:   # the reference's staging errors
        raise _Fail("staging", getattr(exc, "message", str(exc)), getattr(exc, "span", None))


def cmd_run(args) -> int:
    from .errors import RuntimeGraphError, ValidationError
    from .executor import execute
    from .feeds import FeedSyntaxError, format_value, parse_feed
    try:
        feeds = dict(parse_feed(a) for a in args.feed)
    except FeedSyntaxError as exc:
        raise _Fail("staging", exc.message)
    try:
        graph = _load_graph(args.file, args.entry, args.backend, feeds)
    except OSError as exc:
        raise _Fail("usage", f"cannot read {args.file}: {exc.strerror}")
    except SkbError as exc:
        raise _Fail("staging", exc.message, getattr(exc, "span", None))
    try:
        res = execute(graph, feeds, precision=args.precision)
    except (RuntimeGraphError, ValidationError) as exc:
        raise _Fail("runtime", exc.message, getattr(exc, "span", None))
    except SkbError as exc:
        raise _Fail("runtime", exc.message, getattr(exc, "span", None))
    for line in res.print_log:
        print(line)
    for v in res.outputs:
        print(format_value(v))
    return 0


def build_parser() -> _Parser:
    p = _Parser(prog="skb", description="B200 executor for staged control-flow graphs")
    sub = p.add_subparsers(dest="command", required=True)
    r = sub.add_parser("run", help="execute a staged program on the GPU")
    r.add_argument("file")
    r.add_argument("--entry", default="main")
    r.add_argument("--backend", choices=("graph", "sexpr"), default="graph")
    r.add_argument("--feed", "--arg", dest="feed", action="append", default=[], metavar="NAME=SPEC")
    r.add_argument("--precision", choices=("fast", "f64"), default=None)
    r.set_defaults(fn=cmd_run)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except _Fail as f:
        return _report(getattr(args, "file", "<cli>"), f)


if __name__ == "__main__":
    sys.exit(main())
