"""TEST INFRASTRUCTURE ONLY: CPU oracle (see oracle/oracle.py). Never imported by the product."""
