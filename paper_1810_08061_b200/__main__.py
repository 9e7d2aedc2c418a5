"""`python -m paper_1810_08061_b200 run ...` (cli.py)."""
import sys

from .cli import main

sys.exit(main())
