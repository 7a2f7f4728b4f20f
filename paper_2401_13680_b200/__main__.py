"""``python -m paper_2401_13680_b200 <discover|sweep|label|eval> ...`` (see cli.py)."""

from .cli import entry

entry()
