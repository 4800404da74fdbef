"""python -m paper_2502_18738_b200 simulate|bench (see cli.py)."""
from .cli import main

raise SystemExit(main())
