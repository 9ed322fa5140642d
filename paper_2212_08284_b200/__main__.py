"""`python -m paper_2212_08284_b200 {energy,compare,gen,bench}` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
