"""CPU oracle for the SageSched hot path -- TEST INFRASTRUCTURE ONLY.

Importable only by tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs; the product package never imports it.
"""
