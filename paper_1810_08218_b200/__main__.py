"""`python -m paper_1810_08218_b200 ...`: the command-line front end (cli.py)."""
import sys

from .cli import main

sys.exit(main())
