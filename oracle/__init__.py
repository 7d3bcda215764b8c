"""TEST INFRASTRUCTURE ONLY: parity oracle (see oracle/oracle.py). Never imported by the product."""
