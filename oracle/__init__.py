"""ORACLE — test infrastructure only (CPU restatement of the reference path).
Never imported by the product package."""
