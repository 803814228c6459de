"""Camera matrices for the 3-D density image (host-side plumbing).

The paper's vertex shader applies a Model-View matrix and the geometry shader a View-Projection
(perspective) matrix; the library takes their product as one row-major 4x4 (ff_project, 3 axes).
Conventions: OpenGL lookAt / perspective (right-handed eye space, camera looks down -z), computed in
float64 and rounded once to float32.
"""
import numpy as np


def look_at(eye, target, up):
    eye, target, up = (np.asarray(v, dtype=np.float64) for v in (eye, target, up))
    f = target - eye
    f /= np.linalg.norm(f)
    s = np.cross(f, up)
    s /= np.linalg.norm(s)
    u = np.cross(s, f)
    M = np.eye(4)
    M[0, :3], M[1, :3], M[2, :3] = s, u, -f
    M[:3, 3] = -M[:3, :3] @ eye
    return M


def perspective(fov_y_deg, aspect, near, far):
    f = 1.0 / np.tan(np.radians(fov_y_deg) / 2)
    P = np.zeros((4, 4))
    P[0, 0] = f / aspect
    P[1, 1] = f
    P[2, 2] = (far + near) / (near - far)
    P[2, 3] = 2 * far * near / (near - far)
    P[3, 2] = -1.0
    return P


def view_projection(eye, target, up, fov_y_deg=45.0, aspect=1.0, near=1.0, far=500.0):
    """Row-major float32 4x4 P @ V for ff_project (rows 0, 1, 3 are used)."""
    return (perspective(fov_y_deg, aspect, near, far) @ look_at(eye, target, up)).astype(np.float32)


def lorenz_camera():
    """Config-2 camera: eye (0,-120,25) looking at (0,0,25), up +z, fov 45."""
    return view_projection((0.0, -120.0, 25.0), (0.0, 0.0, 25.0), (0.0, 0.0, 1.0))


def box_camera(lo, hi, eye_dir=(1.6, -2.2, 1.2), fov_y_deg=40.0, aspect=1.0):
    """View-projection that first maps the axis box [lo, hi] (3 axes, possibly of very different
    extents, e.g. (x, y, w_ss) of the STN-GPe bifurcation diagram) onto the unit
    cube centred at the origin, then looks at it from direction `eye_dir` (row-major float32)."""
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    S = np.eye(4)
    S[:3, :3] = np.diag(1.0 / (hi - lo))
    S[:3, 3] = -(lo + hi) / 2 / (hi - lo)
    d = np.asarray(eye_dir, np.float64)
    eye = d / np.linalg.norm(d) * 2.6
    P = perspective(fov_y_deg, aspect, 0.1, 20.0) @ look_at(eye, (0.0, 0.0, 0.0), (0.0, 0.0, 1.0))
    return (P @ S).astype(np.float32)
