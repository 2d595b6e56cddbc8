"""`python -m paper_2512_08321_b200 ...` — the `crtgemm` command line (cli.py)."""
from .cli import main

main()
