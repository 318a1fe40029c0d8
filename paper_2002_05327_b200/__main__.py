"""`python -m paper_2002_05327_b200 <command>` -- the drivers' CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
