"""B200-native PGD-TO optimizer step (arXiv 2511.13905) — drop-in for the
reference's projection / optimizer-step interface."""
from .api import (ConstraintLinearization, DomainError, InfeasibleLinearization,  # noqa: F401
                  NumericalError, ParameterError, PgdSettings, ProjectionOptions,
                  ProjectionPath, ProjectionResult, SingularSystemError, StepResult,
                  UnsupportedProblem, constraint_residual_h, delta_of_y, pgd_step, project,
                  project_general_newton, project_independent, project_single_binary_search,
                  to_string)
from . import synth  # noqa: F401
