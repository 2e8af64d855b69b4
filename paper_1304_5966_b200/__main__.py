"""python -m paper_1304_5966_b200 TARGET.fa QUERY.fa [options] (cli.py)."""
from .cli import main

main()
