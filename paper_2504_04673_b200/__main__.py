"""`python -m paper_2504_04673_b200 ...` runs the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
