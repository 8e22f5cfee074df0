"""python -m paper_1407_7506_b200 ... (cli.py)."""
from .cli import console_main

console_main()
