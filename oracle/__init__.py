"""TEST INFRASTRUCTURE: CPU checkers (C restatement + the compiled reference); see checkers.py."""
