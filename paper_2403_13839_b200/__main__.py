"""`python -m paper_2403_13839_b200 decompile|verify ...` (cli.py)."""
import sys

from .cli import main

sys.exit(main())
