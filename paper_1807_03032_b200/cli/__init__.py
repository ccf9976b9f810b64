"""Command line (spec parser + driver) on the B200 backend."""

from .driver import main, report_text  # noqa: F401
from .spec import ProblemSpec, SpecError, parse_spec, pretty_print  # noqa: F401
