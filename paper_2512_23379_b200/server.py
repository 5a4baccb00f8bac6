"""WebSocket front door over the B200 streaming engine.

Wire protocol of the reference (`pkg/src/ftlk/server.py:1-16`), JSON text
frames both ways:

    client -> server   {"type":"start","seed":u64,"identity":[...],"fps":25}
                       {"type":"drive","index":n,"value":f}
                       {"type":"stop"}
    server -> client   {"type":"frame","index":n,"mouth":f,"state":[...],"chunk":c}
                       {"type":"stats","startup_ms":f,"fps":f,"cycle":{...}}
                       {"type":"error","message":s}

Behaviour kept from the reference: one live stream per connection; malformed
messages get an error message and the socket stays open; the identity is
validated (length, finite, nonzero) and normalised server-side, and the
session's reference frame is `world.P @ identity` (server.py:96-113); a stats
message follows every chunk boundary (server.py:55-71); a session failure is
reported as an error and ends the pump, not the connection.

`world` is any object with `spec.identity_dim`, `P` (D, I) and `mouth(frames)`
(the reference's `World` works as is). The session is this package's
`StreamSession`, so every frame on the wire was denoised by the device engine.
"""

import asyncio
import contextlib
import json

import numpy as np

from .config import SamplerPlan, StreamConfig
from .streaming import StreamSession

WS_PATH = "/ws"


def _dump(kind, **fields):
    return json.dumps(dict(type=kind, **fields))


def frame_message(frame, world):
    mouth = float(np.asarray(world.mouth(np.asarray(frame.state)[None, :]))[0])
    return _dump("frame", index=int(frame.index), mouth=mouth, state=[float(x) for x in np.ravel(frame.state)],
                 chunk=int(frame.chunk))


def stats_message(stats):
    return _dump("stats", startup_ms=float(stats.startup_ms), fps=float(stats.fps),
                 cycle={k: float(v) for k, v in stats.cycle.items()})


def error_message(message):
    return _dump("error", message=str(message))


class _Connection:
    """State of one socket: at most one session and the task pumping its frames."""

    def __init__(self, ws, make_session, world):
        self.ws, self.make_session, self.world = ws, make_session, world
        self.session = None
        self.pump = None

    async def send_error(self, message):
        await self.ws.send_text(error_message(message))

    async def _pump_frames(self):
        sent_chunks = 0
        try:
            while True:
                frames, stats = await asyncio.to_thread(self.session.next_frames, True, 0.1)
                for f in frames:
                    await self.ws.send_text(frame_message(f, self.world))
                if stats.chunks_emitted > sent_chunks:
                    sent_chunks = stats.chunks_emitted
                    await self.ws.send_text(stats_message(stats))
        except asyncio.CancelledError:
            raise
        except Exception as exc:  # noqa: BLE001  (numeric blowups etc.: report, keep the socket)
            with contextlib.suppress(Exception):
                await self.send_error(exc)

    async def on_start(self, msg):
        if self.session is not None:
            return await self.send_error("stream already started")
        try:
            seed = int(msg["seed"])
            identity = np.asarray(msg["identity"], dtype=np.float64)
            fps = float(msg.get("fps", 25.0))
            want = self.world.spec.identity_dim
            if identity.shape != (want,):
                raise ValueError("identity must have %d entries" % want)
            norm = float(np.linalg.norm(identity))
            if not np.isfinite(norm) or norm == 0.0:
                raise ValueError("identity must be finite and nonzero")
            self.session = self.make_session(seed, fps, self.world.P @ (identity / norm))
        except (KeyError, ValueError, TypeError) as exc:
            return await self.send_error("bad start message: %s" % exc)
        self.pump = asyncio.create_task(self._pump_frames())

    async def on_drive(self, msg):
        if self.session is None:
            return await self.send_error("drive before start")
        try:
            sample = (int(msg["index"]), float(msg["value"]))
        except (KeyError, ValueError, TypeError) as exc:
            return await self.send_error("bad drive message: %s" % exc)
        try:
            self.session.push_signal([sample])
        except Exception as exc:  # noqa: BLE001  (ConfigError: out of order, non-finite, closed)
            await self.send_error(exc)

    async def serve(self):
        from starlette.websockets import WebSocketDisconnect
        handlers = {"start": self.on_start, "drive": self.on_drive}
        try:
            while True:
                raw = await self.ws.receive_text()
                try:
                    msg = json.loads(raw)
                except json.JSONDecodeError:
                    await self.send_error("message is not valid JSON")
                    continue
                kind = msg.get("type") if isinstance(msg, dict) else None
                if kind == "stop":
                    break
                handler = handlers.get(kind)
                if handler is None:
                    await self.send_error("unknown message type: %r" % (kind,))
                    continue
                await handler(msg)
        except WebSocketDisconnect:
            pass
        finally:
            await self.shutdown()

    async def shutdown(self):
        if self.pump is not None:
            self.pump.cancel()
            with contextlib.suppress(asyncio.CancelledError):
                await self.pump
        if self.session is not None:
            await asyncio.to_thread(self.session.close)
        with contextlib.suppress(Exception):
            await self.ws.close()


def build_app(store, net_cfg, world, codec, *, sampler=None, chunk_len=9, motion_len=2, pacing="realtime",
              device="cuda"):
    """FastAPI app serving the stream protocol at WS_PATH (reference server.py:74-148)."""
    from fastapi import FastAPI, WebSocket

    plan = sampler if sampler is not None else SamplerPlan()

    def make_session(seed, fps, reference_frame):
        cfg = StreamConfig(chunk_len=chunk_len, motion_len=motion_len, target_fps=fps, sampler=plan, seed=seed,
                           pacing=pacing)
        return StreamSession(store, net_cfg, codec, reference_frame, cfg, device=device)

    app = FastAPI()

    @app.websocket(WS_PATH)
    async def stream_endpoint(ws: WebSocket):
        await ws.accept()
        await _Connection(ws, make_session, world).serve()

    return app


def serve(store, net_cfg, world, codec, *, host="127.0.0.1", port=8787, **app_kwargs):
    """Blocking uvicorn runner (reference server.py:151-159)."""
    import uvicorn
    uvicorn.run(build_app(store, net_cfg, world, codec, **app_kwargs), host=host, port=port, log_level="warning")
