"""TEST INFRASTRUCTURE ONLY: CPU oracle for the signature-kernel path.

May be imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg -- never by the product package.
"""
